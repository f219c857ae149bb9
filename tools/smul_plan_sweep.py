"""Device time of every device-feasible SMUL plan (the reference's candidate list,
bigmul/smul.py:75-105, K a multiple of 32 and <= 32768) for N x N-bit products -- the data
behind smul.device_select_params.  python tools/smul_plan_sweep.py [--bits 16 18 20 ...]"""
import argparse
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_04955_b200._native import SmulDevicePlan  # noqa: E402
from paper_1503_04955_b200.smul import DEVICE_K_MAX, device_select_params, smul_plan_candidates  # noqa: E402
from paper_1503_04955_b200.words import int_to_u32  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, nargs="+", default=[16, 18, 20, 22, 24, 26])
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for e in args.bits:
    N = 1 << e
    r = random.Random(e)
    a, b = r.getrandbits(N) | 1 << (N - 1), r.getrandbits(N) | 1 << (N - 1)
    nl = N // 32
    dA = torch.from_numpy(int_to_u32(a, nl).view(np.int32)).cuda()
    dB = torch.from_numpy(int_to_u32(b, nl).view(np.int32)).cuda()
    chosen = device_select_params(2 * N, 64)
    rows = []
    for p in smul_plan_candidates(2 * N, True, 64):
        if p.K % 32 or p.K > DEVICE_K_MAX or p.n * (p.K // 32) * 4 * 4 > 2 << 30:
            continue
        dp = SmulDevicePlan(p.N, p.m, p.s, p.K, p.omega_exp)
        dC = torch.zeros(dp.product_limbs, dtype=torch.int32, device="cuda")
        run = lambda: dp.mul_device(1, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), dp.product_limbs, s)  # noqa
        run()
        torch.cuda.synchronize()
        ok = int.from_bytes(dC.cpu().numpy().view(np.uint32).tobytes(), "little") == a * b
        ts = []
        for i in range(args.reps + 1):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1))
        rows.append({"m": p.m, "K": p.K, "ms": round(float(np.median(ts)), 4), "exact": ok,
                     "chosen": (p.m, p.K) == (chosen.m, chosen.K)})
        dp.close()
        del dC
    print(json.dumps({"bits": e, "plans": rows}), flush=True)
