"""GPU parity: every stage and every product of the CUDA path (called through the C ABI)
against the reference's golden vectors, the CPU oracle, and Python's int product.
Bit-exact (integer path)."""
import json
import os
import random

import numpy as np
import pytest

from oracle.oracle import OraclePlan
from paper_1503_04955_b200 import Natural, dmul, dmul_many, mul
from paper_1503_04955_b200 import plan as P
from paper_1503_04955_b200.dkss import (device_plan, dkss_decode, dkss_encode, dkss_fft, r_mul, dkss_fft_limbs,
                                        r_mul_limbs)
from paper_1503_04955_b200.words import int_to_u32, u32_to_int, using_word_bits

pytestmark = pytest.mark.gpu


def _stages(golden_dir):
    with open(os.path.join(golden_dir, "stages_index.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("idx", range(7))
def test_stages_equal_reference(cuda_ok, golden_dir, idx):
    r = _stages(golden_dir)[idx]
    g = np.load(os.path.join(golden_dir, f"stages_{r['tag']}.npz"))
    with using_word_bits(r["w"]):
        pl = P.dkss_select_params(r["N"], r["w"])
    dp = device_plan(pl)
    a, b = u32_to_int(g["a"]), u32_to_int(g["b"])
    assert np.array_equal(dp.encode(int_to_u32(a, dp.info["operand_limbs"])), g["enc_a"])
    assert np.array_equal(dp.fft(g["enc_a"]), g["fft_a"])
    assert np.array_equal(dp.fft(np.stack([g["enc_a"], g["enc_b"]])), np.stack([g["fft_a"], g["fft_b"]]))
    assert np.array_equal(dp.rmul(g["fft_a"], g["fft_b"]), g["pointwise"])
    assert np.array_equal(dp.fft(g["pointwise"]), g["fft_c"])
    assert np.array_equal(dp.decode(g["fft_c"], g["product"].size), g["product"])
    prod = dp.mul_limbs(int_to_u32(a, dp.info["operand_limbs"]), int_to_u32(b, dp.info["operand_limbs"]),
                        dp.info["product_limbs"])
    assert np.array_equal(prod[: g["product"].size], g["product"])


@pytest.mark.parametrize("tag", ["m16", "m32"])
def test_rmul_equal_reference(cuda_ok, golden_dir, tag):
    g = np.load(os.path.join(golden_dir, f"rmul_{tag}.npz"))
    m = g["x"].shape[1]
    pl = P.make_plan(1 << 16 if m == 16 else 1 << 24, m, m, u32_to_int(g["p"]), check_bounds=False)
    assert np.array_equal(r_mul_limbs(g["x"], g["y"], pl), g["z"])


def test_reference_list_api(cuda_ok, rng):
    # the reference-shaped stage functions (lists of ints in and out)
    pl = P.dkss_select_params(1 << 12)
    a = rng.getrandbits(4000)
    poly = dkss_encode(a, pl)
    assert len(poly) == 2 * pl.M and all(len(c) == pl.m for c in poly)
    o = OraclePlan(pl)
    want = o.fft(o.encode(a))
    dkss_fft(poly, pl)
    assert poly == [[int.from_bytes(c.tobytes(), "little") for c in row] for row in want]
    x, y = poly[3], poly[7]
    z = r_mul(x, y, pl)
    assert z == P.poly_mul_mod(x, y, pl.m, pl.p)   # schoolbook oracle, tests/test_dkss.py:111-119
    # pipeline x enc(1) is the identity (tests/test_dkss.py:247-260)
    one = dkss_encode(1, pl)
    dkss_fft(one, pl)
    prod = [r_mul(u, v, pl) for u, v in zip(poly, one)]
    dkss_fft(prod, pl)
    assert dkss_decode(prod, pl).to_int() == a


@pytest.mark.parametrize("e", [10, 12, 14, 16, 18, 20])
def test_dmul_powers_of_two(cuda_ok, e):
    rng = random.Random(e)
    N = 1 << e
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N) | 1 << (N - 1)
    assert dmul(a, b) == a * b


def test_dmul_adversarial_all_ones(cuda_ok):
    # config 2b: (2^N - 1)^2, longest carry chains (BASELINE.json configs[1])
    for N in (1 << 16, 1 << 20):
        a = (1 << N) - 1
        assert dmul(a, a) == a * a


def test_dmul_matches_oracle_2_20(cuda_ok):
    rng = random.Random(2)
    N = 1 << 20
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N) | 1 << (N - 1)
    o = OraclePlan(P.dkss_select_params(N))
    assert dmul(a, b).to_int() == o.dmul(a, b) == a * b


def test_dmul_odd_sizes_and_unbalanced(cuda_ok, rng):
    for bits in (1, 31, 1000, 1023, 2049, 3648 * 64 - 5, 99_999):
        a = rng.getrandbits(bits) | 1 << (bits - 1)
        b = rng.getrandbits(max(1, bits // 3) + 1)
        assert dmul(a, b) == a * b
    a = rng.getrandbits(2000 * 64)          # tests/test_dkss.py:284-287
    b = rng.getrandbits(37 * 64)
    assert dmul(Natural.from_int(a), Natural.from_int(b)).to_int() == a * b


def test_dmul_result_length_and_word_sizes(cuda_ok, rng):
    a = Natural.from_int(rng.getrandbits(640), length=12)
    b = Natural.from_int(rng.getrandbits(640), length=10)
    r = dmul(a, b)
    assert len(r) == 22 and r.to_int() == a.to_int() * b.to_int()
    for w, words in ((8, 900), (32, 700)):    # tests/test_dkss.py:292-300
        with using_word_bits(w):
            bits = words * w
            x = rng.getrandbits(bits) | 1 << (bits - 1)
            y = rng.getrandbits(bits) | 1 << (bits - 1)
            assert dmul(Natural.from_int(x, length=words), Natural.from_int(y, length=words)).to_int() == x * y


def test_mul_routes_dmul(cuda_ok, rng):
    a, b = rng.getrandbits(600 * 64), rng.getrandbits(600 * 64)
    assert mul(a, b, algorithm="dmul") == a * b
    from paper_1503_04955_b200 import ThresholdTable

    # tests/test_bench.py:24-30: 600-word inputs routed to dmul by the table
    assert mul(a, b, thresholds=ThresholdTable(kmul=4, t3mul=16, smul=128, dmul=512)) == a * b


def test_plan_info_op_counts(cuda_ok):
    # ring products per multiply == the reference's ks_calls (bigmul/dkss.py:412)
    for e, (rf, tot) in {16: (465, 1907), 20: (14849, 52739)}.items():
        dp = device_plan(P.dkss_select_params(1 << e))
        assert dp.info["twiddles_per_fft"] == rf and dp.info["ring_products"] == tot


def test_batched_products(cuda_ok):
    # config 3 shape (smaller batch): pair i from Random(seed0 + i)
    pairs = []
    for i in range(64):
        r = random.Random(3 + i)
        N = 1 << 18
        pairs.append((r.getrandbits(N) | 1 << (N - 1), r.getrandbits(N) | 1 << (N - 1)))
    got = dmul_many(pairs)
    assert got == [a * b for a, b in pairs]


def test_pipelined_batch_ragged(cuda_ok):
    # >= 64 pairs run as 8 chunks on two device lanes (dkss._pipelined_batch): uneven chunk
    # sizes, ragged operand lengths, all-ones pairs, results in input order
    rng = random.Random(21)
    pairs = []
    for i in range(131):
        na, nb = rng.randrange(1, 1 << 16), rng.randrange(1, 1 << 16)
        pairs.append((rng.getrandbits(na) | 1, rng.getrandbits(nb) | 1))
    pairs[7] = pairs[100] = ((1 << (1 << 16)) - 1, (1 << (1 << 16)) - 1)
    got = dmul_many(pairs)
    assert [g.to_int() for g in got] == [a * b for a, b in pairs]
    assert dmul_many(pairs[:3]) == [a * b for a, b in pairs[:3]]  # below the pipelining threshold


def test_device_api_graph_replay(cuda_ok):
    import torch

    N = 1 << 18
    pl = P.dkss_select_params(N)
    dp = device_plan(pl)
    nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
    rng = random.Random(9)
    pairs = [(rng.getrandbits(N), rng.getrandbits(N)) for _ in range(4)]
    A = torch.from_numpy(np.stack([int_to_u32(a, nl) for a, _ in pairs]).view(np.int32)).cuda()
    B = torch.from_numpy(np.stack([int_to_u32(b, nl) for _, b in pairs]).view(np.int32)).cuda()
    C = torch.zeros((4, npl), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for rep in range(3):   # first call captures the CUDA graph, later calls replay it
        C.zero_()
        dp.mul_device(4, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), npl, s)
        torch.cuda.synchronize()
        out = C.cpu().numpy().view(np.uint32)
        assert [u32_to_int(row) for row in out] == [a * b for a, b in pairs]
    prof = dp.profile_device(4, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), s)
    kinds = [k for k, *_ in prof]
    levels_in_passes = 1 if "rows" in kinds else pl.levels  # DKSS_ROWS=1: levels >= 1 run in k_rows
    assert kinds.count("fwd_pass") == levels_in_passes and kinds.count("inv_pass") == levels_in_passes
    assert all(ms > 0 for _, ms, _, _ in prof)


def test_errors_are_reported(cuda_ok):
    pl = P.dkss_select_params(1 << 12)
    dp = device_plan(pl)
    with pytest.raises(ValueError):
        dp.encode(int_to_u32(1 << 5000, 200))      # operand >= 2^N (bigmul/dkss.py:389-390)
    with pytest.raises(ValueError):
        dp.mul_limbs(int_to_u32((1 << 4096) - 1, 128), int_to_u32((1 << 4096) - 1, 128), 10)  # nc too small


@pytest.mark.slow
def test_dmul_2_24(cuda_ok):
    rng = random.Random(4)
    N = 1 << 24
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N) | 1 << (N - 1)
    c = dmul(a, b).to_int()
    # residue check (cheap) plus the full product
    for q in (2**61 - 1, 2**62 - 57, 2**59 - 55):
        assert c % q == (a % q) * (b % q) % q
    assert c == a * b


def test_dmul_2_26_residues(cuda_ok):
    # config 5: checked by residues modulo 64 seeded random 62-bit primes (BASELINE.json configs[4])
    from paper_1503_04955_b200.numtheory import lucas_prime_test, factor_smooth

    rng = random.Random(5)
    N = 1 << 26
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N) | 1 << (N - 1)
    c = dmul(a, b).to_int()
    assert c.bit_length() in (2 * N - 1, 2 * N)
    pr = random.Random(12345)
    primes = []
    while len(primes) < 64:
        q = pr.getrandbits(62) | 1 << 61 | 1
        if all(pow(w, q - 1, q) == 1 for w in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)):
            primes.append(q)
    for q in primes:
        assert c % q == (a % q) * (b % q) % q


# --- four-step split of one multiply, G ranks emulated on one GPU ---------
@pytest.mark.parametrize("dist_decode", [True, False])
@pytest.mark.parametrize("e,world", [(16, 2), (16, 16), (18, 4), (20, 2), (20, 8), (20, 32)])
def test_fourstep_virtual_ranks(cuda_ok, e, world, dist_decode):
    from paper_1503_04955_b200.fourstep import dmul_fourstep_virtual

    rng = random.Random(100 + e + world)
    N = 1 << e
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N) | 1 << (N - 1)
    assert dmul_fourstep_virtual(a, b, world, distributed_decode=dist_decode) == a * b


@pytest.mark.parametrize("e,world", [(18, 4), (20, 2), (20, 8), (22, 4), (24, 8), (24, 32)])
def test_fourstep_virtual_fused_exchange(cuda_ok, e, world):
    # the exchange fused into the phase kernels' stores (dkss_fs_*_peer), emulated ranks' buffers
    # as the peer table: equal to a*b and to the all-to-all path
    from paper_1503_04955_b200.fourstep import dmul_fourstep_virtual

    rng = random.Random(300 + e + world)
    N = 1 << e
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N) | 1 << (N - 1)
    c = dmul_fourstep_virtual(a, b, world, exchange="peer")
    if e <= 22:
        assert c == a * b
    else:
        assert c == dmul_fourstep_virtual(a, b, world)
        for q in (2**61 - 1, 2**62 - 57, 2**59 - 55):
            assert c % q == (a % q) * (b % q) % q
    ones = (1 << N) - 1
    if e <= 20:
        assert dmul_fourstep_virtual(ones, ones, world, exchange="peer") == ones * ones


def test_fourstep_virtual_all_ones(cuda_ok):
    from paper_1503_04955_b200.fourstep import dmul_fourstep_virtual

    N = 1 << 20
    a = (1 << N) - 1
    assert dmul_fourstep_virtual(a, a, 4) == a * a


def test_fourstep_virtual_2_24_matches_single_gpu(cuda_ok):
    from paper_1503_04955_b200.fourstep import dmul_fourstep_virtual

    rng = random.Random(4)
    N = 1 << 24
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N) | 1 << (N - 1)
    c = dmul_fourstep_virtual(a, b, 8)
    assert c == dmul(a, b).to_int()
    for q in (2**61 - 1, 2**62 - 57):
        assert c % q == (a % q) * (b % q) % q


def test_fourstep_rejects_bad_world(cuda_ok):
    pl = P.dkss_select_params(1 << 20)
    dp = device_plan(pl)
    for world in (3, 64, 0):
        with pytest.raises(ValueError):
            dp.fs_layout(world)


@pytest.mark.parametrize("digit_bits", [8, 13, 16, 30, 32])
def test_mul_digits_radix(cuda_ok, digit_bits):
    # dkss_mul_digits: operands as radix-2^k digit strings (k = 30 is CPython's int digit)
    rng = random.Random(digit_bits)
    pl = P.dkss_select_params(1 << 16)
    dp = device_plan(pl)
    a, b = rng.getrandbits(1 << 16), rng.getrandbits((1 << 16) - 77)
    mask = (1 << digit_bits) - 1
    da = np.array([(a >> (digit_bits * i)) & mask for i in range(-(-a.bit_length() // digit_bits) + 3)], np.uint32)
    db = np.array([(b >> (digit_bits * i)) & mask for i in range(-(-b.bit_length() // digit_bits))], np.uint32)
    c = dp.mul_digits(da.ctypes.data, da.size, db.ctypes.data, db.size, digit_bits, dp.info["product_limbs"])
    assert u32_to_int(c) == a * b
    if digit_bits < 32:
        bad = da.copy()
        bad[0] = 1 << digit_bits
        with pytest.raises(ValueError):
            dp.mul_digits(bad.ctypes.data, bad.size, db.ctypes.data, db.size, digit_bits, dp.info["product_limbs"])


def test_dmul_chain_natural_operands(cuda_ok, rng):
    # a lazy Natural product fed back as an operand takes the 32-bit limb route
    a, b, c = rng.getrandbits(20000), rng.getrandbits(30000), rng.getrandbits(50000)
    ab = dmul(a, b)
    abc = dmul(ab, c)
    assert abc.to_int() == a * b * c and len(abc) == len(ab) + -(-c.bit_length() // 64)
    assert dmul(c, Natural.from_int(a)).to_int() == a * c


# --- row phase in one cluster kernel (k_rows): every two-level plan size, multiply and square
@pytest.mark.parametrize("e", [18, 19, 21, 22, 23])
def test_dmul_two_level_plans(cuda_ok, e):
    rng = random.Random(500 + e)
    N = 1 << e
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N - 3)
    assert dmul(a, b).to_int() == a * b
    assert dmul(a, a).to_int() == a * a  # squaring mode (same object -> one forward transform)


def test_square_batch_and_all_ones(cuda_ok):
    rng = random.Random(9)
    xs = [rng.getrandbits(1 << 18) for _ in range(5)] + [(1 << (1 << 18)) - 1]
    got = dmul_many([(x, x) for x in xs])
    assert [g.to_int() for g in got] == [x * x for x in xs]


@pytest.mark.parametrize("row_phase,pass_kind,twiddle", [
    ("persistent", "auto", "cuda"), ("launches", "auto", "cuda"), ("cluster", "auto", "cuda"),
    ("launches", "warp", "cuda"), ("launches", "split", "cuda"), ("auto", "cta", "cuda"),
    ("auto", "auto", "tensor"), ("auto", "auto", "auto")])
def test_kernel_shape_variants(cuda_ok, row_phase, pass_kind, twiddle):
    # every kernel shape a plan can be built with (include/dkss.h dkss_plan_opts) gives the same
    # products: two-level sizes of both inner lengths, squares and a batch
    from paper_1503_04955_b200._native import DevicePlan
    from paper_1503_04955_b200.dkss import plan_capacity

    r = random.Random(11)
    for e in (18, 20, 21, 23):
        N = 1 << e
        pl = P.dkss_select_params(N)
        dp = DevicePlan(plan_capacity(pl), pl.M, pl.m, pl.u, pl.p, pl.rho_powers, 0, row_phase=row_phase,
                        pass_kind=pass_kind, twiddle=twiddle)
        nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
        a, b = r.getrandbits(N), r.getrandbits(N)
        A, B = int_to_u32(a, nl), int_to_u32(b, nl)
        assert u32_to_int(dp.mul_limbs(A, B, npl)) == a * b, e
        sq = dp.mul_digits(A.ctypes.data, nl, A.ctypes.data, nl, 32, npl)  # same pointers: squaring mode
        assert u32_to_int(sq) == a * a, e
        if e == 18:
            ps = [(r.getrandbits(N), r.getrandbits(N)) for _ in range(6)]
            C = dp.mul_batch(np.stack([int_to_u32(x, nl) for x, _ in ps]), np.stack([int_to_u32(y, nl) for _, y in ps]))
            assert [u32_to_int(c) for c in C] == [x * y for x, y in ps]
        dp.close()


def test_plans_and_graphs_do_not_leak(cuda_ok):
    # 1000 plan create/destroy cycles and 100 distinct device-buffer triples (one cached CUDA
    # graph each, LRU-capped per plan): device memory stays bounded
    import torch

    from paper_1503_04955_b200._native import DevicePlan
    from paper_1503_04955_b200.dkss import plan_capacity

    pl = P.dkss_select_params(1 << 12)
    args = (plan_capacity(pl), pl.M, pl.m, pl.u, pl.p, pl.rho_powers, 0)
    torch.cuda.init()
    # one plan and one multiply first: the kernels' code is loaded lazily at their first launch
    # and must not count as a leak when this test runs before any other multiply of this shape
    warm = DevicePlan(*args)
    wl, wp = warm.info["operand_limbs"], warm.info["product_limbs"]
    wa = torch.zeros(wl, dtype=torch.int32, device="cuda")
    wc = torch.zeros(wp, dtype=torch.int32, device="cuda")
    warm.mul_device(1, wa.data_ptr(), wa.data_ptr(), wl, wc.data_ptr(), wc.numel())
    torch.cuda.synchronize()
    warm.close()
    del wa, wc
    torch.cuda.empty_cache()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(1000):
        DevicePlan(*args).close()
    dp = DevicePlan(*args)
    nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
    dev = torch.device("cuda", 0)
    r = random.Random(5)
    for i in range(100):
        a, b = r.getrandbits(4000), r.getrandbits(4000)
        A = torch.from_numpy(int_to_u32(a, nl).view(np.int32)).to(dev)
        B = torch.from_numpy(int_to_u32(b, nl).view(np.int32)).to(dev)
        C = torch.zeros(npl + i % 3, dtype=torch.int32, device=dev)
        dp.mul_device(1, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), C.numel())
        torch.cuda.synchronize()
        assert u32_to_int(C.cpu().numpy().view(np.uint32)) == a * b
        del A, B, C
    dp.close()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20, (free0, free1)


@pytest.mark.parametrize("e", [27, 28])
def test_dmul_beyond_the_configs_residues(cuda_ok, e):
    # SURVEY.md 8(f) "general plans": N >= 2^27 selects d = 192 (L = 6 limbs) and u = 64;
    # 2^28 needs three column levels.  Checked by residues modulo 32 seeded 62-bit primes.
    rng = random.Random(e)
    N = 1 << e
    a = rng.getrandbits(N) | 1 << (N - 1)
    b = rng.getrandbits(N) | 1 << (N - 1)
    pl = P.dkss_select_params(N)
    assert -(-pl.p.bit_length() // 32) == 6 and pl.u == 64
    c = dmul(a, b).to_int()
    assert c.bit_length() in (2 * N - 1, 2 * N)
    pr = random.Random(777)
    primes = []
    while len(primes) < 32:
        q = pr.getrandbits(62) | 1 << 61 | 1
        if all(pow(w, q - 1, q) == 1 for w in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)):
            primes.append(q)
    for q in primes:
        assert c % q == (a % q) * (b % q) % q


@pytest.mark.parametrize("e", [16, 18, 20, 22, 24])
def test_tensor_core_twiddles_match_cuda_cores(cuda_ok, e):
    # the same transform with the table twiddles on the tensor cores (tcgen05 kind::i8, dkss_tc.cuh)
    # and on the CUDA cores (IMAD.WIDE ring_mul): identical stage outputs and products
    from paper_1503_04955_b200._native import DevicePlan
    from paper_1503_04955_b200.dkss import plan_capacity

    N = 1 << e
    pl = P.dkss_select_params(N)
    mk = lambda tw: DevicePlan(plan_capacity(pl), pl.M, pl.m, pl.u, pl.p, pl.rho_powers, 0, twiddle=tw)  # noqa: E731
    tcp, cup = mk("tensor"), mk("cuda")
    rng = random.Random(e)
    nl, npl = tcp.info["operand_limbs"], tcp.info["product_limbs"]
    a, b = rng.getrandbits(N) | 1 << (N - 1), rng.getrandbits(N) | 1 << (N - 1)
    ea = tcp.encode(int_to_u32(a, nl))
    assert np.array_equal(tcp.fft(ea), cup.fft(ea))
    if e <= 20:
        o = OraclePlan(pl)
        assert np.array_equal(tcp.fft(ea), o.fft(ea))
    A, B = int_to_u32(a, nl), int_to_u32(b, nl)
    c = tcp.mul_limbs(A, B, npl)
    assert np.array_equal(c, cup.mul_limbs(A, B, npl))
    assert u32_to_int(c) == a * b
    ones = int_to_u32((1 << N) - 1, nl)
    assert u32_to_int(tcp.mul_limbs(ones, ones, npl)) == ((1 << N) - 1) ** 2
    tcp.close()
    cup.close()


def test_dmul_without_cpython_digit_layout(cuda_ok, rng, monkeypatch):
    # the e2e path's fallback when the interpreter's int layout is not the checked one: operands
    # go to the C ABI as 32-bit limbs (int_to_u32) instead of CPython's 30-bit digits
    from paper_1503_04955_b200 import words

    monkeypatch.setattr(words, "_PYLONG_OK", False)
    for e in (12, 20, 24):
        a = rng.getrandbits(1 << e) | 1 << ((1 << e) - 1)
        b = rng.getrandbits((1 << e) - 7) | 1
        assert dmul(a, b).to_int() == a * b
