"""Golden vectors for the SMUL path, produced by the REFERENCE implementation (this container only).

The reference (/root/reference/pkg/src/bigmul, pure Python) is imported read-only; every
number written here comes from its own functions (smul_select_params, smul_plan_candidates,
bit_slices, shuffle_indices, fft_eval over FermatRing, _cyclic_coeff_product, smul).

Outputs
  tests/golden/smul_plans.json   outermost plans (and candidate counts) for a grid of N at w = 64/32/8,
                                 plus plans with a table-forced FFT depth
  tests/golden/smul_stages.npz   for three small outermost plans: the shuffled slices of a,
                                 their forward fft_eval, the inverse fft_eval of a vector holding
                                 0, 2^K and random residues, the normalised cyclic coefficient
                                 product of a and b, and a*b

usage: PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_smul.py
"""

import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

import importlib  # noqa: E402

S = importlib.import_module("bigmul.smul")
from bigmul.basecase import ThresholdTable  # noqa: E402
from bigmul.fermat import FermatRing  # noqa: E402
from bigmul.fft import fft_eval, shuffle_indices  # noqa: E402
from bigmul.words import Natural, ScratchArena, bit_slices, using_word_bits  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def plan_dict(p):
    return {"N": p.N, "m": p.m, "n": p.n, "s": p.s, "K": p.K, "omega_exp": p.omega_exp,
            "theta_exp": p.theta_exp, "outermost": p.outermost, "w": p.w}


def elems(v, K):
    kw = K // 32
    x = np.zeros((len(v), kw), dtype=np.uint32)
    top = np.zeros(len(v), dtype=np.uint32)
    for i, val in enumerate(v):
        top[i] = val >> K
        x[i] = np.frombuffer((val & ((1 << K) - 1)).to_bytes(4 * kw, "little"), dtype=np.uint32)
    return x, top


def main():
    plans = []
    sizes = sorted({1 << e for e in range(9, 28)} | {3 << e for e in range(9, 25)} | {1000, 4097, 12345, 99999})
    for w in (64, 32, 8):
        with using_word_bits(w):
            for N in sizes:
                p = S.smul_select_params(N, outermost=True, w=w)
                plans.append({"n0": N, "w": w, "plan": plan_dict(p),
                              "candidates": len(S.smul_plan_candidates(N, True, w))})
    forced = []
    for N, m in ((1 << 20, 10), (1 << 21, 13), (3 << 18, 11)):
        t = ThresholdTable()
        t.smul_fft_m[max(0, (N // 64).bit_length() - 1)] = m
        forced.append({"n0": N, "w": 64, "m": m, "plan": plan_dict(S.smul_select_params(N, True, 64, t))})
    with open(os.path.join(OUT, "smul_plans.json"), "w") as f:
        json.dump({"plans": plans, "forced": forced}, f, indent=0)

    rng = random.Random(1503)
    arrays = {}
    index = []
    for tag, n0 in (("n4096", 4096), ("n20000", 20000), ("n131072", 131072)):
        p = S.smul_select_params(n0, outermost=True, w=64)
        a = rng.getrandbits(n0 // 2) | 1 << (n0 // 2 - 1)
        b = rng.getrandbits(n0 - n0 // 2) | 1 << (n0 - n0 // 2 - 1)
        idx = shuffle_indices(p.n)
        av = bit_slices(a, p.s, p.n)
        bv = bit_slices(b, p.s, p.n)
        aw = [av[idx[i]] for i in range(p.n)]
        x, t = elems(aw, p.K)
        arrays[f"{tag}_a_shuffled"], arrays[f"{tag}_a_shuffled_top"] = x, t
        fwd = FermatRing(p.K, p.omega_exp, p.n)
        fft_eval(aw, fwd)
        x, t = elems(aw, p.K)
        arrays[f"{tag}_a_fft"], arrays[f"{tag}_a_fft_top"] = x, t
        mod = (1 << p.K) + 1
        v = [rng.randrange(mod) for _ in range(p.n)]
        v[0], v[1], v[-1] = 0, 1 << p.K, 1 << p.K
        x, t = elems(v, p.K)
        arrays[f"{tag}_v"], arrays[f"{tag}_v_top"] = x, t
        fft_eval(v, fwd.inverse_ring())
        x, t = elems(v, p.K)
        arrays[f"{tag}_v_inv"], arrays[f"{tag}_v_inv_top"] = x, t
        arena = ScratchArena()
        cv = S._cyclic_coeff_product(av, bv, p, ThresholdTable(), arena)
        x, t = elems(cv, p.K)
        arrays[f"{tag}_coeffs"], arrays[f"{tag}_coeffs_top"] = x, t
        prod = S.smul(Natural.from_int(a), Natural.from_int(b)).to_int()
        assert prod == a * b
        nl = -(-n0 // 32)
        arrays[f"{tag}_a"] = np.frombuffer(a.to_bytes(4 * nl, "little"), dtype=np.uint32).copy()
        arrays[f"{tag}_b"] = np.frombuffer(b.to_bytes(4 * nl, "little"), dtype=np.uint32).copy()
        arrays[f"{tag}_prod"] = np.frombuffer(prod.to_bytes(8 * nl, "little"), dtype=np.uint32).copy()
        index.append({"tag": tag, "n0": n0, "plan": plan_dict(p)})
    np.savez_compressed(os.path.join(OUT, "smul_stages.npz"), **arrays)
    with open(os.path.join(OUT, "smul_stages_index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print("wrote", len(plans), "plans,", len(index), "stage sets")


if __name__ == "__main__":
    main()
