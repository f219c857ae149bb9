"""Generate golden vectors by running the REFERENCE implementation (this container only).

The reference (/root/reference/pkg/src/bigmul, pure Python) is imported read-only
and its own functions produce every number written here; nothing in this repo's
package is used.  The GPU box never sees /root/reference -- tests there read
only the fixtures this script commits under tests/golden/.

Outputs
  tests/golden/plans.json        plan fields for N = 2^10..2^26 (+ paper rows) at w = 64/32/8
  tests/golden/stages_<tag>.npz  stage vectors for small real plans:
                                 encode(a), encode(b), dkss_fft(a), dkss_fft(b),
                                 pointwise r_mul, dkss_fft(c), decode -> product limbs
  tests/golden/rmul_<tag>.npz    r_mul(x, y) on random canonical inputs (m = 16, 32)
  tests/golden/ref_tests.json    known-answer vectors from the reference test-suite

usage: PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py
"""

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from bigmul import dkss as R  # noqa: E402
from bigmul.basecase import ThresholdTable  # noqa: E402
from bigmul.numtheory import modinv  # noqa: E402
from bigmul.words import Natural, ScratchArena, using_word_bits  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")
FAST = ThresholdTable(kmul=16, t3mul=64, smul=2500)


def limbs(poly, L):
    """list[2M][m] of ints -> uint32[2M, m, L]"""
    n = len(poly)
    m = len(poly[0])
    raw = b"".join(c.to_bytes(4 * L, "little") for row in poly for c in row)
    return np.frombuffer(raw, dtype=np.uint32).reshape(n, m, L).copy()


def rho_hash(plan):
    h = hashlib.sha256()
    for s in range(plan.mu):
        for k in range(plan.m):
            h.update(plan.rho_powers[s][k].to_bytes(16 if plan.d <= 128 else 32, "little"))
    return h.hexdigest()[:16]


def plan_record(N, w):
    with using_word_bits(w):
        t = time.time()
        plan = R.dkss_select_params(N, w)
        dt = time.time() - t
    rec = dict(N=N, w=w, M=plan.M, m=plan.m, u=plan.u, p=str(plan.p), d=plan.d, zeta=plan.zeta,
               omega=str(plan.omega), gamma=str(plan.gamma), inv2M=str(modinv(2 * plan.M, plan.p)),
               rho=[str(c) for c in plan.rho], rho_sha=rho_hash(plan), ks_stride=plan.ks_stride,
               iclen=plan.iclen, oclen=plan.oclen, trace=R.plan_trace(plan), build_s=round(dt, 3))
    if plan.mu <= 64:
        rec["rho_powers"] = [[str(c) for c in row] for row in plan.rho_powers]
    return rec


def stages(tag, N, w, seed, all_ones=False):
    with using_word_bits(w):
        plan = R.dkss_select_params(N, w)
        L = -(-plan.d // 32)
        rng = random.Random(seed)
        if all_ones:
            a = b = (1 << N) - 1
        else:
            a = rng.getrandbits(N) | 1 << (N - 1)
            b = rng.getrandbits(N) | 1 << (N - 1)
        ar = ScratchArena()
        ea = R.dkss_encode(Natural.from_int(a), plan, ar)
        eb = R.dkss_encode(Natural.from_int(b), plan, ar)
        fa = [list(x) for x in ea]
        fb = [list(x) for x in eb]
        plan.ks_calls = 0
        R.dkss_fft(fa, plan, FAST, ar)
        fft_calls = plan.ks_calls
        R.dkss_fft(fb, plan, FAST, ar)
        pw = [R.r_mul(x, y, plan, FAST, ar) for x, y in zip(fa, fb)]
        ic = [list(x) for x in pw]
        R.dkss_fft(ic, plan, FAST, ar)
        prod = R.dkss_decode(ic, plan, ar).to_int()
        assert prod == a * b
        nlimb = -(-2 * N // 32)
        np.savez_compressed(
            os.path.join(OUT, f"stages_{tag}.npz"),
            a=np.frombuffer(a.to_bytes(4 * (-(-N // 32)), "little"), dtype=np.uint32),
            b=np.frombuffer(b.to_bytes(4 * (-(-N // 32)), "little"), dtype=np.uint32),
            enc_a=limbs(ea, L), enc_b=limbs(eb, L), fft_a=limbs(fa, L), fft_b=limbs(fb, L),
            pointwise=limbs(pw, L), fft_c=limbs(ic, L),
            product=np.frombuffer(prod.to_bytes(4 * nlimb, "little"), dtype=np.uint32),
            meta=np.array([N, w, plan.M, plan.m, plan.u, L, seed, int(all_ones), fft_calls], dtype=np.int64),
            p=np.frombuffer(plan.p.to_bytes(4 * L, "little"), dtype=np.uint32))
        return dict(tag=tag, N=N, w=w, M=plan.M, m=plan.m, u=plan.u, L=L, seed=seed, fft_calls=fft_calls)


def rmul_vectors(tag, m, count, seed):
    p = R.proth_table()[128][0]
    plan = R.make_plan(0, m, m, p, check_bounds=False)
    rng = random.Random(seed)
    xs = [[rng.randrange(p) for _ in range(m)] for _ in range(count)]
    ys = [[rng.randrange(p) for _ in range(m)] for _ in range(count)]
    # include edge values: zeros, p-1 everywhere, identity
    xs[0] = [p - 1] * m
    ys[0] = [p - 1] * m
    xs[1] = [0] * m
    ys[2] = [1] + [0] * (m - 1)
    zs = [R.r_mul(x, y, plan, FAST) for x, y in zip(xs, ys)]
    np.savez_compressed(os.path.join(OUT, f"rmul_{tag}.npz"), x=limbs(xs, 4), y=limbs(ys, 4), z=limbs(zs, 4),
                        p=np.frombuffer(p.to_bytes(16, "little"), dtype=np.uint32))


def ref_test_vectors():
    """Known answers that the reference's own tests pin (tests/test_dkss.py)."""
    out = {}
    # tests/test_dkss.py:55-57
    out["omega_193_64_5"] = R.find_root_omega(193, 64, 5)
    # tests/test_dkss.py:67-82
    om = R.find_root_omega(17, 8, 3)
    out["rho_17_4_2"] = R.compute_rho(17, 4, 2, om)[0]
    # tests/test_dkss.py:94-101
    out["xpow_17"] = {str(e): R.poly_mul_xpow([1, 2, 3, 4], e, 4, 17) for e in range(8)}
    # tests/test_dkss.py:130-135
    plan = R.make_plan(0, 4, 2, 17, check_bounds=False)
    v = [[3, 5], [7, 11]]
    R.dkss_inner_fft_eval(v, plan)
    out["butterfly_17"] = v
    # toy plans' rho (tests/test_dkss.py:85-91)
    out["toy_rho"] = {f"{M},{m},{p}": R.make_plan(0, M, m, p, check_bounds=False).rho
                      for M, m, p in [(4, 2, 17), (8, 2, 17), (8, 4, 97), (16, 4, 97)]}
    # paper rows (tests/test_dkss.py:303-310)
    pl = R.dkss_select_params(3648 * 64, w=64)
    out["paper_3648"] = [pl.M, pl.m, pl.iclen, pl.u]
    M, m, u, p, g = R.select_geometry(42991616 * 64, w=64)
    out["paper_42991616"] = [M, m, u, str(p), g]
    # dkss_fft / r_mul on the toy plans the reference tests use (tests/test_dkss.py:185-202, :111-119)
    rng = random.Random(0xC0FFEE)
    toy = []
    for M, m, p in [(2, 2, 17), (4, 2, 17), (8, 2, 17), (8, 4, 97), (16, 4, 97)]:
        plan = R.make_plan(0, M, m, p, check_bounds=False)
        vals = [[rng.randrange(p) for _ in range(m)] for _ in range(2 * M)]
        work = [list(v) for v in vals]
        R.dkss_fft(work, plan, FAST)
        xs = [[rng.randrange(p) for _ in range(m)] for _ in range(8)]
        ys = [[rng.randrange(p) for _ in range(m)] for _ in range(8)]
        zs = [R.r_mul(x, y, plan, FAST) for x, y in zip(xs, ys)]
        toy.append(dict(M=M, m=m, p=p, rho_powers=plan.rho_powers, fft_in=vals, fft_out=work, x=xs, y=ys, z=zs))
    out["toy_plans"] = toy
    return out


def proth_digest():
    """sha256 of the reference prime table's (bits, h, g) records (bigmul/data/proth_primes.txt)."""
    rows = R.proth_table()
    text = "\n".join(f"{bits} {h} {g}" for bits, (p, h, g) in sorted(rows.items()))
    return {"rows": len(rows), "sha256": hashlib.sha256(text.encode()).hexdigest()}


def main():
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "proth_digest.json"), "w") as f:
        json.dump(proth_digest(), f)
    t0 = time.time()
    plans = []
    for w in (64, 32, 8):
        for e in range(10, 27):
            plans.append(plan_record(1 << e, w))
    for N in (1000, 1500, 3000, 3648 * 64, 7168 * 64, 12345, 99999, 777777):
        plans.append(plan_record(N, 64))
    with open(os.path.join(OUT, "plans.json"), "w") as f:
        json.dump(plans, f, indent=0)
    print(f"plans: {len(plans)} in {time.time() - t0:.1f}s", flush=True)

    with open(os.path.join(OUT, "ref_tests.json"), "w") as f:
        json.dump(ref_test_vectors(), f, indent=0)

    rmul_vectors("m16", 16, 64, 11)
    rmul_vectors("m32", 32, 32, 12)
    print(f"rmul done {time.time() - t0:.1f}s", flush=True)

    meta = []
    meta.append(stages("n4096_w64", 4096, 64, 3))          # m=16, L=2, u=16
    meta.append(stages("n3000_w64", 3000, 64, 4))          # non power of 2, u=24
    meta.append(stages("n65536_w64", 1 << 16, 64, 1))      # config 1 plan (m=16, L=4)
    meta.append(stages("n65536_w32", 1 << 16, 32, 5))      # d=96 -> L=3
    meta.append(stages("n65536_w8", 1 << 16, 8, 6))        # d=80 -> L=3
    meta.append(stages("n65536_ones", 1 << 16, 64, 0, all_ones=True))
    meta.append(stages("n1500_w64", 1500, 64, 7))          # m=8
    print(f"stages done {time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(OUT, "stages_index.json"), "w") as f:
        json.dump(meta, f, indent=0)


if __name__ == "__main__":
    main()
