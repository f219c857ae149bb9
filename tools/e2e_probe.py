"""End-to-end pieces of dmul(int, int) at one size: the host-buffer C call with a pinned product
buffer (direct D2H) and with an ordinary one (staging copy), plus raw PCIe copies for scale.

  python tools/e2e_probe.py [--bits 24] [--reps 10]
"""
import argparse
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_04955_b200._native import pinned_empty  # noqa: E402
from paper_1503_04955_b200.dkss import _hot_plan, dmul  # noqa: E402
from paper_1503_04955_b200.words import pylong_digits  # noqa: E402


def med(f, reps):
    f()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return round(ts[len(ts) // 2] * 1e6, 1)


ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=24)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
N = 1 << args.bits
r = random.Random(4)
a = r.getrandbits(N) | 1 << (N - 1)
b = r.getrandbits(N) | 1 << (N - 1)
plan, dp, nl, npl, fp, rp = _hot_plan(N, 64)
(pa, na), (pb, nb) = pylong_digits(a), pylong_digits(b)
bits = 30 | 0x100
out = {}
out["dmul_us"] = med(lambda: dmul(a, b), args.reps)
out["mul_digits_pinned_out_us"] = med(lambda: dp.mul_digits(pa, na, pb, nb, bits, npl), args.reps)


def pageable():
    c = np.empty(npl, dtype=np.uint32)
    dp._check_call = dp._lib.dkss_mul_digits(dp._h, pa, na, pb, nb, bits, c.ctypes.data, npl)


import ctypes  # noqa: E402

dp._lib.dkss_mul_digits.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
out["mul_digits_pageable_out_us"] = med(pageable, args.reps)
h = pinned_empty((npl,))
d = torch.empty(npl, dtype=torch.int32, device="cuda")
ht = torch.from_numpy(h.view(np.int32))
out["d2h_pinned_us"] = med(lambda: (ht.copy_(d, non_blocking=True), torch.cuda.synchronize()), args.reps)
out["h2d_pinned_us"] = med(lambda: (d.copy_(ht, non_blocking=True), torch.cuda.synchronize()), args.reps)
out["product_bytes"] = 4 * npl
print(out)
