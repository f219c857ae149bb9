"""The GPU dmul registered into the REFERENCE package and driven by the reference's own callers.

``paper_1503_04955_b200.integration.install`` puts the device dmul into ``bigmul``'s plugin table
and the names ``mul`` calls directly (bigmul/dispatch.py:11-46).  Then, unmodified reference code
runs it: ``mul`` (forced by name and by the threshold ladder), ``run_bench`` +
``quotient_column`` (bigmul/bench.py:42-91), ``lucas_lehmer(p, "dmul")`` (bigmul/bench.py:197-217)
and the checks of the reference's own DKSS tests (tests/test_dkss.py:278-300,
tests/test_bench.py:24-39) and memory criterion (tests/test_acceptance.py:183-206).

Two device backends:
* ``stub`` (CPU suite): the device plan is replaced by a Python stand-in that reads the operand
  digits the host code hands to the C ABI and multiplies them with Python ints, so every host-side
  step of the drop-in (operand types, word sizes, digit staging, result class and length, arena)
  runs without a GPU;
* ``gpu`` (``-m gpu``): the real libdkss on the device.

The reference is imported from ``baseline/_ref`` (the offline install the bench contract allows,
shipped to the GPU box) or, in the build container, ``/root/reference/pkg/src``.
"""
import ctypes
import importlib
import os
import random
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PATHS = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def _import_reference():
    for path in REF_PATHS:
        if os.path.isdir(os.path.join(path, "bigmul")):
            if path not in sys.path:
                sys.path.insert(0, path)
            os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
            sys.dont_write_bytecode = True
            return importlib.import_module("bigmul")
    pytest.skip("reference package not available (baseline/_ref or /root/reference)")


class StubDevicePlan:
    """Stands in for _native.DevicePlan on a machine without a GPU: same constructor and the
    product entry points dmul / dmul_many use; the digits are read from the host addresses the
    host code passes, exactly as the C ABI reads them."""

    def __init__(self, N, M, m, u, p, rho_powers, device=0, row_phase="auto", pass_kind="auto", **_):
        from paper_1503_04955_b200._native import footprint_bytes

        L = -(-p.bit_length() // 32)
        self.N = N
        self.info = {"operand_limbs": -(-N // 32), "product_limbs": -(-2 * N // 32), "L": L,
                     "poly_bytes": 2 * M * m * L * 4, "footprint_bytes": footprint_bytes(N, M, m, L)}
        self.calls = 0

    skip_products_above = None  # bits; the memory test only needs the arena at its largest size

    @staticmethod
    def _value(addr, n, bits):
        from paper_1503_04955_b200.words import join_bits

        if n == 0:
            return 0
        return join_bits((ctypes.c_uint32 * n).from_address(addr), bits & 0xFF)

    def _limbs(self, v, nc):
        if v >> (32 * nc):
            raise ValueError("product does not fit")
        return np.frombuffer(v.to_bytes(4 * nc, "little"), dtype=np.uint32).copy()

    def mul_digits(self, pa, na, pb, nb, bits, nc):
        a, b = self._value(pa, na, bits), self._value(pb, nb, bits)
        if max(a.bit_length(), b.bit_length()) > self.N:
            raise ValueError("operand does not fit the plan")
        self.calls += 1
        if self.skip_products_above and a.bit_length() > self.skip_products_above:
            return np.zeros(nc, dtype=np.uint32)
        return self._limbs(a * b, nc)

    def mul_limbs(self, A, B, nc):
        self.calls += 1
        return self._limbs(int.from_bytes(A.tobytes(), "little") * int.from_bytes(B.tobytes(), "little"), nc)

    def mul_batch_digits(self, pas, nas, pbs, nbs, bits, nc, out=None):
        C = np.stack([self.mul_digits(pa, na, pb, nb, bits, nc) for pa, na, pb, nb in zip(pas, nas, pbs, nbs)])
        if out is not None:
            out[...] = C
            return out
        return C

    def mul_batch(self, A, B, nc=None):
        nc = nc or self.info["product_limbs"]
        return np.stack([self.mul_limbs(a, b, nc) for a, b in zip(A, B)])

    def close(self):
        pass


@pytest.fixture(params=["stub", pytest.param("gpu", marks=pytest.mark.gpu)])
def ref(request, monkeypatch):
    """The reference package with the B200 dmul installed (stubbed device or the real one)."""
    from paper_1503_04955_b200 import dkss
    from paper_1503_04955_b200.integration import install

    bigmul = _import_reference()
    if request.param == "stub":
        monkeypatch.setattr(dkss, "DevicePlan", StubDevicePlan)
    else:
        import torch

        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    dkss.clear_device_plans()
    undo = install(bigmul)
    yield bigmul
    undo()
    StubDevicePlan.skip_products_above = None
    dkss.clear_device_plans()


def test_install_rebinds_table_and_names(ref):
    from paper_1503_04955_b200 import dkss

    from bigmul import dispatch
    assert dispatch.dmul is ref.dmul and dispatch.dmul.__module__ == "paper_1503_04955_b200.integration"
    a = ref.words.Natural.from_int(3)
    # the table entry and the name both reach the GPU dmul (the reference's own dmul is untouched)
    got = dispatch.ALGORITHMS["dmul"](a, a, None, ref.words.ScratchArena())
    assert type(got) is ref.words.Natural and got.to_int() == 9 and len(got) == 2
    assert sys.modules["bigmul.dkss"].dmul is not dispatch.dmul
    assert dkss._dev_plans  # a device plan was built for it


def test_reference_dkss_tests_with_gpu_dmul(ref):
    """tests/test_dkss.py:278-300 of the reference, with its dmul replaced."""
    from bigmul.basecase import ThresholdTable
    from bigmul.smul import smul as ref_smul
    from bigmul.words import Natural, using_word_bits

    dmul = ref.dispatch.dmul
    FAST = ThresholdTable(kmul=16, t3mul=64, smul=2500)
    rng = random.Random(0xC0FFEE)
    a = Natural.from_int(0xDEAD, length=2)
    assert dmul(a, Natural.from_int(1)) == a
    assert dmul(a, Natural.from_int(0)).to_int() == 0
    assert len(dmul(a, Natural.from_int(0))) == 3
    for words in (300, 1000):
        bits = words * 64
        x = rng.getrandbits(bits) | 1 << (bits - 1)
        y = rng.getrandbits(bits) | 1 << (bits - 1)
        na, nb = Natural.from_int(x, length=words), Natural.from_int(y, length=words)
        got = dmul(na, nb, FAST)
        assert got == ref_smul(na, nb, FAST)  # the reference's own equality (bigmul.words.Natural)
        assert type(got) is Natural and len(got) == 2 * words
    x, y = rng.getrandbits(2000 * 64), rng.getrandbits(37 * 64)
    assert dmul(Natural.from_int(x), Natural.from_int(y), FAST).to_int() == x * y
    with using_word_bits(8):  # the reference's 8-bit build: plan and words at w = 8
        for words in (400, 900):
            bits = words * 8
            x = rng.getrandbits(bits) | 1 << (bits - 1)
            y = rng.getrandbits(bits) | 1 << (bits - 1)
            got = dmul(Natural.from_int(x, length=words), Natural.from_int(y, length=words), FAST)
            assert got.to_int() == x * y and len(got) == 2 * words
            assert all(0 <= w < 256 for w in got.words)


def test_reference_mul_dispatch(ref):
    """tests/test_bench.py:24-39 of the reference: threshold dispatch reaching dmul, forced names."""
    from bigmul.basecase import ThresholdTable
    from bigmul.dispatch import ALGORITHMS, mul
    from bigmul.words import Natural

    rng = random.Random(7)
    table = ThresholdTable(kmul=4, t3mul=16, smul=128, dmul=512)
    for words in (1, 3, 8, 20, 70, 200, 600, 700):
        x = rng.getrandbits(words * 64) | 1 << (words * 64 - 1)
        y = rng.getrandbits(words * 64) | 1 << (words * 64 - 1)
        got = mul(Natural.from_int(x, length=words), Natural.from_int(y, length=words), table)
        assert got.to_int() == x * y
    x, y = rng.getrandbits(256), rng.getrandbits(256)
    for name in ALGORITHMS:
        assert mul(Natural.from_int(x), Natural.from_int(y), ThresholdTable(kmul=16, t3mul=64, smul=2500),
                   algorithm=name).to_int() == x * y
    with pytest.raises(ValueError):
        mul(Natural.from_int(x), Natural.from_int(y), algorithm="nope")


def test_reference_mul_threshold_reaches_gpu(ref):
    from paper_1503_04955_b200 import dkss

    from bigmul.basecase import ThresholdTable
    from bigmul.dispatch import mul
    from bigmul.words import Natural

    dkss.clear_device_plans()
    x = random.Random(3).getrandbits(600 * 64)
    got = mul(Natural.from_int(x), Natural.from_int(x + 1), ThresholdTable(kmul=4, t3mul=16, smul=128, dmul=512))
    assert got.to_int() == x * (x + 1)
    assert dkss._dev_plans, "the threshold ladder did not reach the GPU dmul"


def test_reference_run_bench_and_quotient(ref):
    """run_bench checks every timed product against its reference algorithm (bigmul/bench.py:57-68)."""
    import io

    from bigmul.bench import quotient_column, run_bench, write_csv

    recs = run_bench(["dmul", "t3mul"], [64, 256], reps=3, seed=89, reference="t3mul")
    assert [(r.algorithm, r.input_words) for r in recs] == [("dmul", 64), ("t3mul", 64), ("dmul", 256),
                                                           ("t3mul", 256)]
    assert all(r.peak_arena_words > 0 for r in recs if r.algorithm == "dmul")
    col = quotient_column(recs, "dmul", "t3mul")
    assert len(col) == 2 and all(q > 0 for _, q in col)
    out = io.StringIO()
    write_csv(recs, out)
    assert out.getvalue().splitlines()[0] == "algorithm,input_words,reps,median_ns,peak_arena_words"


def test_reference_lucas_lehmer_with_gpu_dmul(ref):
    """bigmul/bench.py:197-217: the system test, one squaring per step through ALGORITHMS["dmul"]."""
    from bigmul.bench import lucas_lehmer

    for p, prime in ((61, True), (127, True), (89, True), (67, False), (101, False)):
        got = lucas_lehmer(p, "dmul")
        assert got == lucas_lehmer(p, "t3mul")
        assert got[0] is prime


def test_reference_memory_criterion_dmul(ref):
    """tests/test_acceptance.py:183-206 (criterion 6), the dmul half: the arena peak the GPU dmul
    records (its device footprint: dkss_footprint_bytes) against the published DMUL memory table,
    within the criterion's 15%."""
    from bigmul.words import Natural, ScratchArena

    StubDevicePlan.skip_products_above = 1 << 22  # (stub only) no 2^23-bit Python products
    targets = {3648: 803584, 28160: 6439936, 221184: 51422464}
    rng = random.Random(66)
    for words, want in targets.items():
        x = rng.getrandbits(words * 64) | 1 << (words * 64 - 1)
        y = rng.getrandbits(words * 64) | 1 << (words * 64 - 1)
        arena = ScratchArena()
        got = ref.dispatch.dmul(Natural.from_int(x, length=words), Natural.from_int(y, length=words), None, arena)
        peak = arena.peak_bytes(64)
        assert abs(peak - want) <= 0.15 * want, (words, peak, want)
        if words <= 28160:
            assert got.to_int() == x * y
