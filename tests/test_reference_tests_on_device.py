"""The reference's OWN DKSS tests (tests/test_dkss.py of bigmul) run against the device stages.

The reference test module is loaded from ``baseline/_ref/reference_tests`` (tools/install_reference.sh
copies it next to the offline install) or ``/root/reference/pkg/tests``, and its module globals
``dkss_encode``, ``dkss_fft``, ``r_mul``, ``dkss_decode`` and ``dmul`` are rebound to this package's
device-backed functions -- the test bodies themselves run unmodified.

Device-targetable tests (every plan they build is a real planner plan or a ring with m in
{8, 16, 32} and a multi-limb prime):
  test_r_mul_larger_ring, test_encode_shapes, test_encode_decode_roundtrip_by_evaluation,
  test_dkss_pipeline_toy_roundtrip, test_coefficient_bound_instrumented, test_dmul_identity_zero,
  test_dmul_matches_smul, test_dmul_unbalanced, test_dmul_small_word_build.
Oracle-only tests: test_poly_mul_xpow, test_r_mul_identity_and_schoolbook,
test_dkss_fft_bottom_case_is_inner_fft, test_dkss_fft_matches_naive_evaluation and
test_twiddle_cost_one_ring_product_each use toy rings (m = 2 or 4, p = 17 or 97: one limb); the
device kernels exist for m in {8, 16, 32} and 2..6 limbs (every plan the reference planner emits
for N >= 1024), so the device REFUSES those rings with ValueError -- checked here, so
no toy test can pass on a silent host fallback.  Their algorithm is covered by the oracle
(tests/test_oracle_golden.py replays the same toy vectors).
"""
import importlib.util
import inspect
import os
import random
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DEVICE_TESTS = ["test_r_mul_larger_ring", "test_encode_shapes", "test_encode_decode_roundtrip_by_evaluation",
                "test_dkss_pipeline_toy_roundtrip", "test_coefficient_bound_instrumented", "test_dmul_identity_zero",
                "test_dmul_matches_smul", "test_dmul_unbalanced", "test_dmul_small_word_build"]
ORACLE_ONLY = ["test_poly_mul_xpow", "test_r_mul_identity_and_schoolbook", "test_dkss_fft_bottom_case_is_inner_fft",
               "test_dkss_fft_matches_naive_evaluation", "test_twiddle_cost_one_ring_product_each"]


@pytest.fixture(scope="module")
def ref_test_dkss():
    from test_reference_callers import _import_reference

    _import_reference()
    for d in (os.path.join(ROOT, "baseline", "_ref", "reference_tests"), "/root/reference/pkg/tests"):
        path = os.path.join(d, "test_dkss.py")
        if os.path.exists(path):
            break
    else:
        pytest.skip("reference tests not available (run tools/install_reference.sh)")
    spec = importlib.util.spec_from_file_location("bigmul_reference_test_dkss", path)
    mod = importlib.util.module_from_spec(spec)
    sys.dont_write_bytecode = True
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture
def on_device(ref_test_dkss, monkeypatch, cuda_ok):
    import paper_1503_04955_b200.dkss as dev
    from bigmul.words import set_word_bits

    for name in ("dkss_encode", "dkss_fft", "r_mul", "dkss_decode", "dmul"):
        monkeypatch.setattr(ref_test_dkss, name, getattr(dev, name))
    set_word_bits(64)  # the reference conftest's autouse fixture
    yield ref_test_dkss
    set_word_bits(64)


def _call(fn):
    kw = {}
    for p in inspect.signature(fn).parameters:
        if p == "rng":
            kw[p] = random.Random(0xC0FFEE)  # the reference conftest's rng fixture
        else:
            raise AssertionError(f"unexpected fixture {p}")
    return fn(**kw)


@pytest.mark.parametrize("name", DEVICE_TESTS)
def test_reference_dkss_test_on_device(on_device, name):
    # the stage functions have no host fallback: a test body that passes ran on the device
    _call(getattr(on_device, name))


@pytest.mark.parametrize("name", ORACLE_ONLY)
def test_toy_ring_tests_are_refused_by_the_device(on_device, name):
    with pytest.raises(ValueError):
        _call(getattr(on_device, name))
