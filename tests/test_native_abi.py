"""The C-ABI library loads and exports every symbol include/dkss.h and include/smul.h
declare (no compute: runs on CPU-only machines)."""
import os
import re

from paper_1503_04955_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("dkss.h", "smul.h"):
        with open(os.path.join(ROOT, "include", h)) as f:
            src = f.read()
        names |= set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+((?:dkss|smul)_\w+)\s*\(", src, re.M))
    return sorted(names)


def test_header_declares_expected_entry_points():
    names = _declared()
    assert names == sorted(_native.EXPORTS), names


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.dkss_version() >= 1


def test_structs_match_header_layout():
    import ctypes

    assert ctypes.sizeof(_native.PlanDesc) == 8 + 4 * 4 + 2 * 8
    assert ctypes.sizeof(_native.PlanInfo) >= 8 * 7 + 4 * 7
    assert ctypes.sizeof(_native.SmulPlanDesc) == 8 + 4 + 4 + 8 + 4 + 4  # include/smul.h, padded


def test_bad_plan_options_rejected_before_any_device_work():
    import ctypes

    import numpy as np

    from paper_1503_04955_b200.plan import dkss_select_params

    lib = _native.load()
    pl = dkss_select_params(1 << 12)
    L = -(-pl.p.bit_length() // 32)
    p = np.frombuffer(pl.p.to_bytes(4 * L, "little"), dtype=np.uint32).copy()
    rho = np.frombuffer(b"".join(c.to_bytes(4 * L, "little") for row in pl.rho_powers for c in row),
                        dtype=np.uint32).copy()
    desc = _native.PlanDesc(pl.N, pl.M, pl.m, pl.u, L, _native._ptr(p), _native._ptr(rho))
    for opts in (_native.PlanOpts(9, 0, 0), _native.PlanOpts(0, -1, 0), _native.PlanOpts(-1, 0, 0),
                 _native.PlanOpts(0, 0, 7)):
        h = ctypes.c_void_p()
        rc = lib.dkss_plan_create_ex(ctypes.byref(desc), ctypes.byref(opts), 0, ctypes.byref(h))
        assert rc == _native.DKSS_EINVAL and not h.value
        assert b"plan options" in lib.dkss_last_error()


def test_product_library_reads_no_environment_switches():
    # experiment switches (DKSS_EXP_SKIP, DKSS_FWD_KINDS, ...) exist only in DKSS_VARIANT builds
    with open(_native.LIB_PATH, "rb") as f:
        blob = f.read()
    for name in (b"DKSS_EXP_SKIP", b"DKSS_FWD_KINDS", b"DKSS_PASS_MODE", b"DKSS_NO_DYN", b"DKSS_HOST_TIMING",
                 b"DKSS_SMUL_MINCTA", b"DKSS_NO_PDL"):
        assert name not in blob, name


def test_kernel_launch_counter_starts_at_zero_without_gpu_work():
    assert _native.kernel_launches() >= 0
