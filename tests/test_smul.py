"""SMUL, the reference's comparison baseline: plan selection pinned
field for field to the reference's smul_select_params (tests/golden/smul_plans.json, made
by tools/make_golden_smul.py from the reference itself); on the GPU, fft_eval over the
Fermat ring against the reference's transform vectors (tests/golden/smul_stages.npz) and
the full product against a*b."""
import json
import os
import random

import numpy as np
import pytest

from paper_1503_04955_b200 import Natural, mul
from paper_1503_04955_b200.dispatch import ThresholdTable
from paper_1503_04955_b200.smul import (SmulPlan, device_select_params, fft_eval_fermat, smul,
                                        smul_plan_candidates, smul_select_params)
from paper_1503_04955_b200.words import int_to_u32, using_word_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _fields(p: SmulPlan):
    return {"N": p.N, "m": p.m, "n": p.n, "s": p.s, "K": p.K, "omega_exp": p.omega_exp,
            "theta_exp": p.theta_exp, "outermost": p.outermost, "w": p.w}


def test_plans_match_reference():
    g = _load("smul_plans.json")
    assert len(g["plans"]) > 100
    for e in g["plans"]:
        with using_word_bits(e["w"]):
            assert _fields(smul_select_params(e["n0"], True, e["w"])) == e["plan"], e
            assert len(smul_plan_candidates(e["n0"], True, e["w"])) == e["candidates"], e


def test_forced_depth_matches_reference():
    for e in _load("smul_plans.json")["forced"]:
        t = ThresholdTable()
        t.smul_fft_m[max(0, (e["n0"] // 64).bit_length() - 1)] = e["m"]
        p = smul_select_params(e["n0"], True, 64, t)
        assert _fields(p) == e["plan"]  # a depth with no candidate falls back to the cost model


def test_plan_validation_errors():
    with pytest.raises(ValueError):
        SmulPlan(1001, 3, 8, 125, 1024, 256, 0, True, 64).validate()  # N != s * n
    with pytest.raises(ValueError):
        SmulPlan(1024, 3, 8, 128, 192, 48, 0, True, 64).validate()    # K below m + 2s + 1


@pytest.mark.parametrize("e", range(9, 30, 2))
def test_device_plans_are_valid_candidates(e):
    p = device_select_params(1 << e, 64)
    assert p.K % 32 == 0 and p.K <= 32768 and p.N >= 1 << e
    assert p in smul_plan_candidates(1 << e, True, 64)


# ---- GPU ------------------------------------------------------------------------------

def _elems(x, top, K):
    return [int.from_bytes(x[i].tobytes(), "little") | (int(top[i]) << K) for i in range(len(top))]


def _stage_sets():
    return _load("smul_stages_index.json")


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(3))
def test_fft_matches_reference(cuda_ok, idx):
    e = _stage_sets()[idx]
    p = SmulPlan(**e["plan"])
    z = np.load(os.path.join(GOLD, "smul_stages.npz"))
    t = e["tag"]
    v = _elems(z[f"{t}_a_shuffled"], z[f"{t}_a_shuffled_top"], p.K)
    fft_eval_fermat(v, p)
    assert v == _elems(z[f"{t}_a_fft"], z[f"{t}_a_fft_top"], p.K)
    v = _elems(z[f"{t}_v"], z[f"{t}_v_top"], p.K)  # holds 0 and 2^K
    fft_eval_fermat(v, p, inverse=True)
    assert v == _elems(z[f"{t}_v_inv"], z[f"{t}_v_inv_top"], p.K)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(3))
def test_product_on_reference_plan(cuda_ok, idx):
    from paper_1503_04955_b200._native import SmulDevicePlan

    e = _stage_sets()[idx]
    p = e["plan"]
    z = np.load(os.path.join(GOLD, "smul_stages.npz"))
    t = e["tag"]
    dp = SmulDevicePlan(p["N"], p["m"], p["s"], p["K"], p["omega_exp"])
    prod = z[f"{t}_prod"]
    c = dp.mul_limbs(z[f"{t}_a"].copy(), z[f"{t}_b"].copy(), prod.size)
    assert np.array_equal(c, prod)


@pytest.mark.gpu
def test_smul_equals_product(cuda_ok):
    rng = random.Random(7)
    for bits in (1, 31, 32, 33, 100, 511, 512, 4096, 20000, 65537, 1 << 18, 1 << 20):
        a = rng.getrandbits(bits) | 1 << (bits - 1)
        b = rng.getrandbits(bits) | 1 << (bits - 1)
        assert smul(a, b).to_int() == a * b, bits
        c = rng.getrandbits(max(1, bits // 5)) | 1
        assert smul(a, c).to_int() == a * c, bits  # unbalanced
        assert smul(a, a).to_int() == a * a, bits  # square


@pytest.mark.gpu
@pytest.mark.parametrize("e", [23, 25, 26])
def test_smul_large_products_by_residues(cuda_ok, e):
    # product sizes 2^24, 2^26, 2^27 bits: the Q = 8 / 16 / 32 lane widths of the FFT and
    # pointwise kernels, the CTA-wide (FULL) variants, and a non-full Q = 32 plan (the odd
    # operand length below); checked by residues modulo 62-bit primes, as the DKSS 2^26 test
    from paper_1503_04955_b200.smul import device_plan_for

    rng = random.Random(100 + e)
    for bits in (1 << e, (1 << e) - 12345):
        a = rng.getrandbits(bits) | 1 << (bits - 1)
        b = rng.getrandbits(bits) | 1 << (bits - 1)
        plan, _ = device_plan_for(2 * bits, 64)
        c = smul(a, b).to_int()
        assert c.bit_length() in (2 * bits - 1, 2 * bits), (bits, plan.K)
        pr = random.Random(54321)
        for _ in range(16):
            q = pr.getrandbits(62) | 1 << 61 | 1
            assert c % q == (a % q) * (b % q) % q, (bits, plan.K, q)


@pytest.mark.gpu
def test_smul_edge_values(cuda_ok):
    for bits in (64, 3000, 1 << 16, 1 << 21):
        ones = (1 << bits) - 1                       # longest carry chains
        assert smul(ones, ones).to_int() == ones * ones
        assert smul(1 << (bits - 1), 1 << (bits - 1)).to_int() == 1 << (2 * bits - 2)
        assert smul(ones, 1).to_int() == ones
    r = smul(Natural.from_int(0, length=4), 12345)
    assert r.to_int() == 0 and len(r) == 5


@pytest.mark.gpu
def test_smul_result_length_and_routing(cuda_ok):
    rng = random.Random(11)
    a = Natural.from_int(rng.getrandbits(6400), length=120)
    b = Natural.from_int(rng.getrandbits(6400), length=101)
    r = mul(a, b, algorithm="smul")
    assert len(r) == 221 and r.to_int() == a.to_int() * b.to_int()
    for w in (8, 32):
        with using_word_bits(w):
            x = rng.getrandbits(5000 * w // 8) | 1
            y = rng.getrandbits(4000 * w // 8) | 1
            assert smul(x, y).to_int() == x * y


@pytest.mark.gpu
def test_smul_device_batch(cuda_ok):
    import torch

    from paper_1503_04955_b200.smul import device_plan_for

    rng = random.Random(3)
    bits, batch = 1 << 16, 8
    p, dp = device_plan_for(2 * bits, 64)
    nl = bits // 32
    A = [rng.getrandbits(bits) for _ in range(batch)]
    B = [rng.getrandbits(bits) for _ in range(batch)]
    da = torch.from_numpy(np.stack([int_to_u32(x, nl) for x in A]).view(np.int32)).cuda()
    db = torch.from_numpy(np.stack([int_to_u32(x, nl) for x in B]).view(np.int32)).cuda()
    nc = dp.product_limbs
    dc = torch.zeros(batch, nc, dtype=torch.int32, device="cuda")
    dp.mul_device(batch, da.data_ptr(), db.data_ptr(), nl, dc.data_ptr(), nc, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    C = dc.cpu().numpy().view(np.uint32)
    for i in range(batch):
        assert int.from_bytes(C[i].tobytes(), "little") == A[i] * B[i]
    dp.mul_device(batch, da.data_ptr(), 0, nl, dc.data_ptr(), nc, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    C = dc.cpu().numpy().view(np.uint32)
    assert all(int.from_bytes(C[i].tobytes(), "little") == A[i] * A[i] for i in range(batch))


@pytest.mark.gpu
def test_smul_range_errors(cuda_ok):
    from paper_1503_04955_b200._native import SmulDevicePlan

    dp = SmulDevicePlan(4096, 3, 512, 1088, 272)
    a = int_to_u32((1 << 3000) - 1, 94)
    with pytest.raises(ValueError):
        dp.mul_limbs(a, a, 200)  # 6000-bit product does not fit N = 4096
    with pytest.raises(ValueError):
        SmulDevicePlan(4096, 3, 512, 1080, 270)  # K not a multiple of 32


@pytest.mark.gpu
def test_harness_quotient_dmul_over_smul(cuda_ok):
    import io

    # the REFERENCE's harness (bigmul/bench.py:42-91) with both GPU rungs installed in its table
    from test_reference_callers import _import_reference

    from paper_1503_04955_b200.integration import install

    bigmul = _import_reference()
    from bigmul.bench import quotient_column, run_bench, write_csv

    undo = install(bigmul, smul=True)
    try:
        recs = run_bench(["dmul", "smul"], [64, 1024], reps=3, seed=5, reference="t3mul")
    finally:
        undo()
    assert {(r.algorithm, r.input_words) for r in recs} == {(a, s) for a in ("dmul", "smul") for s in (64, 1024)}
    q = quotient_column(recs)  # T_DMUL / T_SMUL (bigmul/bench.py:80-91)
    assert [s for s, _ in q] == [64, 1024] and all(v > 0 for _, v in q)
    buf = io.StringIO()
    write_csv(recs, buf)
    assert buf.getvalue().count("smul,") == 2


@pytest.mark.gpu
def test_lucas_lehmer_with_smul(cuda_ok):
    from paper_1503_04955_b200.lucas import lucas_lehmer, lucas_lehmer_host

    for p in (521, 607, 1279):  # Mersenne prime exponents
        assert lucas_lehmer(p, "smul") == (True, 0)
    for p in (523, 1277):       # composite 2^p - 1: residue64 as Python's int loop
        assert lucas_lehmer(p, "smul") == lucas_lehmer_host(p)


@pytest.mark.gpu
def test_smul_digits_entry_point(cuda_ok):
    from paper_1503_04955_b200.smul import device_plan_for

    rng = random.Random(13)
    a, b = rng.getrandbits(90000) | 1, rng.getrandbits(70001) | 1
    _, dp = device_plan_for(a.bit_length() + b.bit_length(), 64)

    def digits(x, k):
        return np.array([(x >> (k * i)) & ((1 << k) - 1) for i in range(-(-x.bit_length() // k))], dtype=np.uint32)

    nc = -(-(a.bit_length() + b.bit_length()) // 32)
    for k in (8, 30, 32):  # radix 2^k digit strings, repacked on the device
        da, db = digits(a, k), digits(b, k)
        c = dp.mul_digits(da.ctypes.data, da.size, db.ctypes.data, db.size, k, nc)
        assert int.from_bytes(c.tobytes(), "little") == a * b
    bad = digits(a, 30)
    bad[5] |= 1 << 30  # a digit above 30 bits is rejected unless the caller vouches for it
    with pytest.raises(ValueError):
        dp.mul_digits(bad.ctypes.data, bad.size, bad.ctypes.data, bad.size, 30, nc)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(3))
def test_stage_pipeline_matches_reference_coefficients(cuda_ok, idx):
    # _cyclic_coeff_product (bigmul/smul.py:256-271) composed from the device transforms:
    # slices -> shuffle -> forward fft_eval (GPU) -> pointwise mod 2^K+1 -> shuffle ->
    # inverse fft_eval (GPU) -> 2^-m; equals the reference's normalised coefficients
    from paper_1503_04955_b200.words import bit_slices

    e = _stage_sets()[idx]
    p = SmulPlan(**e["plan"])
    z = np.load(os.path.join(GOLD, "smul_stages.npz"))
    t = e["tag"]
    a = int.from_bytes(z[f"{t}_a"].tobytes(), "little")
    b = int.from_bytes(z[f"{t}_b"].tobytes(), "little")
    idxs = [int(bin(i)[2:].zfill(p.m)[::-1], 2) for i in range(p.n)]
    mod = (1 << p.K) + 1
    av, bv = bit_slices(a, p.s, p.n), bit_slices(b, p.s, p.n)
    aw = [av[idxs[i]] for i in range(p.n)]
    bw = [bv[idxs[i]] for i in range(p.n)]
    fft_eval_fermat(aw, p)
    fft_eval_fermat(bw, p)
    cw = [x * y % mod for x, y in zip(aw, bw)]
    cv = [cw[idxs[i]] for i in range(p.n)]
    fft_eval_fermat(cv, p, inverse=True)
    inv = pow(2, -p.m, mod)
    got = [x * inv % mod for x in cv]
    assert got == _elems(z[f"{t}_coeffs"], z[f"{t}_coeffs_top"], p.K)
