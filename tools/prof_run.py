"""Minimal driver for ncu / compute-sanitizer / experiment libraries: a few device multiplies of
one config through dkss_profile_device, per-kind device time printed (no timing claims: the
launches are not graphed).  With DKSS_LIB pointing at an experiment build the product may be
wrong; the check is reported, not asserted.

usage: python tools/prof_run.py [config] [reps]     (config names as in bench.py)
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
from paper_1503_04955_b200.dkss import device_plan  # noqa: E402
from paper_1503_04955_b200.plan import dkss_select_params  # noqa: E402
from paper_1503_04955_b200.words import int_to_u32, u32_to_int  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "mul2^24"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    N, batch, seed, ones = bench.CONFIGS[cfg]
    pairs = [bench.operand_pair(N, seed, i, ones) for i in range(batch)]
    dp = device_plan(dkss_select_params(N))
    nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
    A = torch.from_numpy(np.stack([int_to_u32(a, nl) for a, _ in pairs]).view(np.int32)).cuda()
    B = torch.from_numpy(np.stack([int_to_u32(b, nl) for _, b in pairs]).view(np.int32)).cuda()
    C = torch.zeros((batch, npl), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    per = {}
    for r in range(reps):
        flush.zero_()
        run = dp.profile_device(batch, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), s)
        if r == 0:
            continue
        for i, (kind, ms, _, _) in enumerate(run):
            per.setdefault((i, kind), []).append(ms)
    torch.cuda.synchronize()
    got = C.cpu().numpy().view(np.uint32)
    a, b = pairs[0]
    ok = u32_to_int(got[0]) == a * b
    lib = os.environ.get("DKSS_LIB", "libdkss.so")
    print(f"{cfg} lib={os.path.basename(lib)} product_ok={ok}")
    for (i, kind), v in sorted(per.items()):
        print(f"  {i:2d} {kind:12s} {1e3 * float(np.median(v)):9.1f} us")
    print(f"  total {1e3 * sum(float(np.median(v)) for v in per.values()):.1f} us")


if __name__ == "__main__":
    main()
