"""Does pinning the CPython int's own digit buffer (cudaHostRegister) beat copying it into a
page-locked staging buffer before the H2D?  One 2^24-bit operand (2.24 MB of 30-bit digits).

  python tools/hostreg_probe.py [--bits 24] [--reps 10]
"""
import argparse
import ctypes
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_04955_b200.words import pylong_digits  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=24)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if rt is None:
    import glob
    rt = ctypes.CDLL(sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[-1])
rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
rt.cudaHostUnregister.argtypes = [ctypes.c_void_p]
rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
N = 1 << args.bits
x = random.Random(1).getrandbits(N) | 1 << (N - 1)
ptr, n = pylong_digits(x)
nbytes = 4 * n
dev = torch.empty(n, dtype=torch.int32, device="cuda")
pin = torch.empty(n, dtype=torch.int32).pin_memory()
src = np.ctypeslib.as_array((ctypes.c_uint32 * n).from_address(ptr))
torch.cuda.synchronize()


def med(f):
    f()
    ts = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e6)
    ts.sort()
    return round(ts[len(ts) // 2], 1)


def staged():
    np.copyto(pin.numpy().view(np.uint32), src)
    rt.cudaMemcpy(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(pin.data_ptr()), nbytes, 1)


def registered():
    base = ptr & ~4095
    size = (ptr + nbytes - base + 4095) & ~4095
    rc = rt.cudaHostRegister(ctypes.c_void_p(base), size, 0)
    if rc:
        raise SystemExit(f"cudaHostRegister rc={rc}")
    rt.cudaMemcpy(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(ptr), nbytes, 1)
    rt.cudaHostUnregister(ctypes.c_void_p(base))


def reg_only():
    base = ptr & ~4095
    size = (ptr + nbytes - base + 4095) & ~4095
    rt.cudaHostRegister(ctypes.c_void_p(base), size, 0)
    rt.cudaHostUnregister(ctypes.c_void_p(base))


def pageable():
    rt.cudaMemcpy(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(ptr), nbytes, 1)


out = {"bytes": nbytes, "staged_copy_h2d_us": med(staged), "register_h2d_unregister_us": med(registered),
       "register_unregister_only_us": med(reg_only), "pageable_h2d_us": med(pageable)}
print(out)
