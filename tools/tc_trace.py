"""Timeline of the tensor-core twiddle kernel's roles on CTA 0 (experiment build with
-DDKSS_TC_TRACE; DKSS_LIB must point at it): per launch, SM-clock stamps of the producer
(stage wait, stage free, copies landed), the MMA thread (full wait, tile ready, per chunk: TMEM
buffer free, chunk issued) and epilogue warp 0 (per chunk: wait, ready, released, stored).

usage: DKSS_LIB=.../libdkss_trace.so python tools/tc_trace.py [config]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
from paper_1503_04955_b200 import _native  # noqa: E402
from paper_1503_04955_b200.dkss import device_plan  # noqa: E402
from paper_1503_04955_b200.plan import dkss_select_params  # noqa: E402
from paper_1503_04955_b200.words import int_to_u32  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "mul2^24"
    N, batch, seed, ones = bench.CONFIGS[cfg]
    pairs = [bench.operand_pair(N, seed, i, ones) for i in range(batch)]
    dp = device_plan(dkss_select_params(N))
    nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
    A = torch.from_numpy(np.stack([int_to_u32(a, nl) for a, _ in pairs]).view(np.int32)).cuda()
    B = torch.from_numpy(np.stack([int_to_u32(b, nl) for _, b in pairs]).view(np.int32)).cuda()
    C = torch.zeros((batch, npl), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        dp.profile_device(batch, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), s)
    torch.cuda.synchronize()
    lib = _native.load()
    buf = np.zeros((8, 3, 512), dtype=np.uint64)
    n = ctypes.c_uint(0)
    rc = lib.dkss_exp_tc_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n))
    assert rc == 0
    print(f"{cfg}: {n.value} tensor-core launches traced; the last four:")
    for slot in [(n.value - 4 + i) % 8 for i in range(4)]:
        tr = buf[slot].astype(np.int64)
        t0 = int(tr[0][0])
        end = int(tr[0][511]) - t0
        def rel(role):
            v = tr[role]
            return [int(x) - t0 for x in v[:511] if x]
        p, m, e = rel(0), rel(1), rel(2)
        print(f"launch slot {slot}: kernel end at {end} clk ({end / 1965:.1f} us)")
        print("  producer (per tile: wait, free, landed):", [tuple(p[1 + 3 * i: 4 + 3 * i]) for i in range((len(p) - 1) // 3)])
        # MMA: start, then per tile: wait, ready, (free, issued) x chunks
        print("  mma:", m)
        print("  epilogue warp 0 (per chunk: wait, ready, released, stored):",
              [tuple(e[1 + 4 * i: 5 + 4 * i]) for i in range((len(e) - 1) // 4)])


if __name__ == "__main__":
    main()
