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
