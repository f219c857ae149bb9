"""Where the end-to-end time of dmul(int, int) goes (host conversion, C-ABI call, device).

  python tools/e2e_breakdown.py [--bits 20] [--reps 50]
"""
import argparse
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_04955_b200.dkss import _plan_for, device_plan, dmul  # noqa: E402
from paper_1503_04955_b200.words import Natural, int_to_u32  # noqa: E402


def med(f, reps):
    f()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return round(ts[len(ts) // 2] * 1e6, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=20)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    N = 1 << args.bits
    r = random.Random(2)
    a = r.getrandbits(N) | 1 << (N - 1)
    b = r.getrandbits(N) | 1 << (N - 1)
    plan = _plan_for(N, 64)
    dp = device_plan(plan)
    nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
    A, B = int_to_u32(a, nl), int_to_u32(b, nl)
    C = dp.mul_limbs(A, B, npl)
    out = {}
    out["dmul_us"] = med(lambda: dmul(a, b), args.reps)
    out["dmul_to_int_us"] = med(lambda: dmul(a, b).to_int(), args.reps)
    out["int_to_u32_x2_us"] = med(lambda: (int_to_u32(a, nl), int_to_u32(b, nl)), args.reps)
    out["c_abi_dkss_mul_us"] = med(lambda: dp.mul_limbs(A, B, npl), args.reps)
    out["natural_from_u32_to_int_us"] = med(lambda: Natural._from_u32(C, 2 * N // 64, 64).to_int(), args.reps)
    dA = torch.from_numpy(A.view(np.int32)).cuda()
    dB = torch.from_numpy(B.view(np.int32)).cuda()
    dC = torch.zeros(npl, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def dev():
        dp.mul_device(1, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), npl, s)
        torch.cuda.synchronize()

    out["device_graph_plus_sync_us"] = med(dev, args.reps)
    hA = torch.from_numpy(A.view(np.int32)).pin_memory()
    hB = torch.from_numpy(B.view(np.int32)).pin_memory()
    hC = torch.empty(npl, dtype=torch.int32).pin_memory()

    def dev_copies():
        dA.copy_(hA, non_blocking=True)
        dB.copy_(hB, non_blocking=True)
        dp.mul_device(1, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), npl, s)
        hC.copy_(dC, non_blocking=True)
        torch.cuda.synchronize()

    out["pinned_h2d_graph_d2h_us"] = med(dev_copies, args.reps)
    out.update(bits=args.bits, operand_bytes=4 * nl, product_bytes=4 * npl)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
