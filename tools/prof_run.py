"""Minimal driver for ncu / compute-sanitizer: a few device multiplies of one config.

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
    cfg = sys.argv[1] if len(sys.argv) > 1 else "mul2^20"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    N, batch, seed, ones = bench.CONFIGS[cfg]
    pairs = bench.operands(N, batch, seed, ones)
    dp = device_plan(dkss_select_params(N))
    nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
    A = torch.from_numpy(np.stack([int_to_u32(a, nl) for a, _ in pairs]).view(np.int32)).cuda()
    B = torch.from_numpy(np.stack([int_to_u32(b, nl) for _, b in pairs]).view(np.int32)).cuda()
    C = torch.zeros((batch, npl), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(reps):
        dp.profile_device(batch, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), s)
    torch.cuda.synchronize()
    got = C.cpu().numpy().view(np.uint32)
    a, b = pairs[0]
    assert u32_to_int(got[0]) == a * b, "product mismatch"
    print("ok", cfg, reps)


if __name__ == "__main__":
    main()
