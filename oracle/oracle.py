"""ctypes front end of the CPU oracle (oracle/dkss_oracle.c).  TEST INFRASTRUCTURE ONLY.

Loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs -- never by the product package.  The oracle is a
C restatement of the reference's DKSS pipeline (bigmul/dkss.py); its parity
with the reference is pinned by tests/test_oracle_golden.py on vectors the
reference produced (tests/golden/).

Arrays are numpy uint32 in the shared layout poly[2M][m][L].
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libdkss_oracle.so")
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(os.path.join(_HERE, "dkss_oracle.c")):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.oracle_plan_create.restype = ctypes.c_void_p
        L.oracle_plan_create.argtypes = [ctypes.c_int] * 5 + [_u32p, _u32p, _u32p]
        L.oracle_plan_destroy.argtypes = [ctypes.c_void_p]
        L.oracle_ks_calls.restype = ctypes.c_longlong
        L.oracle_ks_calls.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_rmul.argtypes = [ctypes.c_void_p, _u32p, _u32p, _u32p, ctypes.c_longlong]
        L.oracle_encode.restype = ctypes.c_int
        L.oracle_encode.argtypes = [ctypes.c_void_p, _u32p, ctypes.c_longlong, _u32p]
        L.oracle_fft.argtypes = [ctypes.c_void_p, _u32p]
        L.oracle_decode.argtypes = [ctypes.c_void_p, _u32p, _u32p, ctypes.c_longlong]
        L.oracle_pointwise.argtypes = [ctypes.c_void_p, _u32p, _u32p, _u32p]
        L.oracle_dmul.restype = ctypes.c_int
        L.oracle_dmul.argtypes = [ctypes.c_void_p, _u32p, ctypes.c_longlong, _u32p, ctypes.c_longlong, _u32p,
                                  ctypes.c_longlong]
        L.oracle_dmul_batch.restype = ctypes.c_int
        L.oracle_dmul_batch.argtypes = [ctypes.c_void_p, ctypes.c_int, _u32p, _u32p, ctypes.c_longlong, _u32p,
                                        ctypes.c_longlong]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(_u32p)


def _limbs(x: int, L: int) -> np.ndarray:
    return np.frombuffer(int(x).to_bytes(4 * L, "little"), dtype=np.uint32).copy()


def set_threads(n: int) -> None:
    lib().oracle_set_threads(n)


def max_threads() -> int:
    return lib().oracle_max_threads()


class OraclePlan:
    """Oracle handle for one host plan (paper_1503_04955_b200.plan.DkssPlan or equivalent)."""

    def __init__(self, plan):
        self.plan = plan
        self.M, self.m, self.u, self.N = plan.M, plan.m, plan.u, plan.N
        self.L = -(-plan.p.bit_length() // 32)
        L = self.L
        p = _limbs(plan.p, L)
        rho = np.concatenate([_limbs(c, L) for row in plan.rho_powers for c in row])
        inv = _limbs(pow(2 * plan.M, -1, plan.p), L)
        self._keep = (p, rho, inv)
        self.h = lib().oracle_plan_create(plan.N, plan.M, plan.m, plan.u, L, _ptr(p), _ptr(rho), _ptr(inv))
        if not self.h:
            raise ValueError("oracle cannot represent this plan")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.oracle_plan_destroy(self.h)
            self.h = None

    @property
    def poly_shape(self):
        return (2 * self.M, self.m, self.L)

    def ks_calls(self, reset=False) -> int:
        return lib().oracle_ks_calls(self.h, int(reset))

    def encode(self, a: int) -> np.ndarray:
        na = max(1, -(-a.bit_length() // 32))
        al = _limbs(a, na)
        out = np.zeros(self.poly_shape, dtype=np.uint32)
        if lib().oracle_encode(self.h, _ptr(al), na, _ptr(out)):
            raise ValueError("operand does not fit the plan")
        return out

    def fft(self, poly: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(poly, dtype=np.uint32).copy()
        lib().oracle_fft(self.h, _ptr(v))
        return v

    def rmul(self, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        y = np.ascontiguousarray(y, dtype=np.uint32)
        out = np.empty_like(x)
        count = x.size // (self.m * self.L)
        lib().oracle_rmul(self.h, _ptr(x), _ptr(y), _ptr(out), count)
        return out

    def decode(self, v: np.ndarray, nout: int) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.uint32)
        out = np.zeros(nout, dtype=np.uint32)
        lib().oracle_decode(self.h, _ptr(v), _ptr(out), nout)
        return out

    def dmul_limbs(self, a: np.ndarray, b: np.ndarray, nout: int) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.zeros(nout, dtype=np.uint32)
        if lib().oracle_dmul(self.h, _ptr(a), a.size, _ptr(b), b.size, _ptr(out), nout):
            raise ValueError("operand does not fit the plan")
        return out

    def dmul(self, a: int, b: int) -> int:
        nl = max(1, -(-max(a.bit_length(), b.bit_length()) // 32))
        nout = 2 * nl
        out = self.dmul_limbs(_limbs(a, nl), _limbs(b, nl), nout)
        return int.from_bytes(out.tobytes(), "little")

    def dmul_batch(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        """a, b: uint32[batch, nlimbs] -> uint32[batch, 2*nlimbs]"""
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        batch, nl = a.shape
        out = np.zeros((batch, 2 * nl), dtype=np.uint32)
        if lib().oracle_dmul_batch(self.h, batch, _ptr(a), _ptr(b), nl, _ptr(out), 2 * nl):
            raise ValueError("operand does not fit the plan")
        return out
