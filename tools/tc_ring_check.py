"""Prototype check + benchmark of the tensor-core twiddle product (tools/tc_ring.cu).

Builds the twiddle's Toeplitz expansion B (s8, balanced base-256 digits of t_l * 2^160 mod p,
negated where the negacyclic product wraps), runs `rows` ring elements through the kernel, checks
every product bit-exactly against the C oracle's r_mul (oracle/dkss_oracle.c, pinned on the
reference's rmul vectors) and reports ring products/s and 32x32 limb-product equivalents/s
(m^2 L^2 per ring product) for comparison with the IMAD.WIDE core
(tools/bench_core.cu, profiles/imad_peak.json).

  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared -Xcompiler -fPIC \
       -o tools/libtc_ring.so tools/tc_ring.cu
  python tools/tc_ring_check.py [--m 16] [--tiles-per-sm 8] [--reps 20]
"""
import argparse
import ctypes
import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import OraclePlan, max_threads, set_threads  # noqa: E402
from paper_1503_04955_b200.plan import dkss_select_params  # noqa: E402

L = 4


def balanced_digits(v: int, nd: int = 17):
    out = []
    for _ in range(nd):
        r = v & 255
        if r >= 128:
            r -= 256
        out.append(r)
        v = (v - r) >> 8
    assert v == 0
    return out


def build_b(t, m, p):
    """B[(j, d)][(i, k)] in the kernel's K-major core layout, N chunks of 256 rows."""
    K, NT = m * 16, m * 32
    T = [(c << 160) % p for c in t]
    dig_pos = [balanced_digits(c) for c in T]
    dig_neg = [balanced_digits(-c) for c in T]
    B = np.zeros((NT, K), dtype=np.int8)
    for j in range(m):
        for i in range(m):
            dg = dig_pos[(j - i) % m] if i <= j else dig_neg[(j - i) % m]
            for kk in range(16):
                for e in range(17):
                    d = kk + e
                    if d < 32:
                        B[j * 32 + d, i * 16 + kk] = dg[e]
                    else:
                        assert dg[e] == 0 or d < 32
    # core layout: chunk of 256 rows n; row n, 16-byte column block c -> (n/8)*SBO + c*128 + (n%8)*16
    sbo = (K // 16) * 128
    out = np.zeros(NT * K, dtype=np.int8)
    for ch in range(NT // 256):
        base = ch * 256 * K
        blk = B[ch * 256:(ch + 1) * 256]
        for n in range(256):
            for c in range(K // 16):
                off = base + (n // 8) * sbo + c * 128 + (n % 8) * 16
                out[off:off + 16] = blk[n, c * 16:(c + 1) * 16]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--tiles-per-sm", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--grid", type=int, default=148)
    args = ap.parse_args()
    m = args.m
    plan = dkss_select_params(1 << 20 if m == 16 else 1 << 24)
    assert plan.m == m
    p = plan.p
    rng = random.Random(7)
    rows = args.grid * 128 * args.tiles_per_sm
    xs = [[rng.randrange(p) for _ in range(m)] for _ in range(rows)]
    xs[0] = [p - 1] * m                       # edges: all p - 1, zero, one
    xs[1] = [0] * m
    xs[2] = [1] + [0] * (m - 1)
    t = [rng.randrange(p) for _ in range(m)]
    X = np.frombuffer(b"".join(c.to_bytes(16, "little") for row in xs for c in row), dtype=np.uint32).copy()
    bm = build_b(t, m, p)
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "libtc_ring.so"))
    lib.tc_ring_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    Z = np.zeros_like(X)
    ms = ctypes.c_float()
    rc = lib.tc_ring_run(m, X.ctypes.data, bm.ctypes.data, Z.ctypes.data, rows, args.reps, args.grid, ctypes.byref(ms))
    if rc:
        raise SystemExit(f"tc_ring_run failed: {rc}")
    set_threads(max_threads())
    o = OraclePlan(plan)
    Xr = X.reshape(rows, m, L)
    Yr = np.broadcast_to(np.frombuffer(b"".join(c.to_bytes(16, "little") for c in t), dtype=np.uint32).reshape(1, m, L),
                         (rows, m, L)).copy()
    want = o.rmul(Xr, Yr)
    got = Z.reshape(rows, m, L)
    bad = np.nonzero(np.any(got != want, axis=(1, 2)))[0]
    rps = rows * args.reps / (ms.value * 1e-3)
    res = {"m": m, "rows": rows, "reps": args.reps, "grid": args.grid, "ms": round(ms.value, 4),
           "ring_products_per_s": round(rps, 0), "limb_product_equiv_per_s": round(rps * m * m * L * L, 0),
           "mismatches": int(bad.size), "first_bad": bad[:5].tolist()}
    print(json.dumps(res))
    if bad.size:
        i = int(bad[0])
        print("row", i, "got", got[i, :2].tolist(), "want", want[i, :2].tolist())
        sys.exit(1)


if __name__ == "__main__":
    main()
