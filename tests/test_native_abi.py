"""The C-ABI library loads and exports every symbol include/dkss.h declares (no compute:
runs on CPU-only machines)."""
import os
import re

from paper_1503_04955_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "dkss.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(dkss_\w+)\s*\(", src, re.M)))


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
