"""Device time of one multiply with the table twiddles on the tensor cores vs the CUDA cores
(same plan, same operands, CUDA-graph replay, L2 flushed before every call) and the per-launch
profile of the tensor-core plan.

  python tools/tc_compare.py [--bits 24] [--batch 1] [--reps 20]
"""
import argparse
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_04955_b200._native import DevicePlan  # noqa: E402
from paper_1503_04955_b200.dkss import plan_capacity  # noqa: E402
from paper_1503_04955_b200.plan import dkss_select_params  # noqa: E402
from paper_1503_04955_b200.words import int_to_u32, u32_to_int  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=24)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
N = 1 << args.bits
pl = dkss_select_params(N)
rng = random.Random(4)
pairs = [(rng.getrandbits(N) | 1 << (N - 1), rng.getrandbits(N) | 1 << (N - 1)) for _ in range(args.batch)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {"bits": args.bits, "batch": args.batch, "plan": {"M": pl.M, "m": pl.m}}
for tw in ("cuda", "tensor"):
    dp = DevicePlan(plan_capacity(pl), pl.M, pl.m, pl.u, pl.p, pl.rho_powers, 0, twiddle=tw)
    nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
    A = torch.from_numpy(np.stack([int_to_u32(a, nl) for a, _ in pairs]).view(np.int32)).cuda()
    B = torch.from_numpy(np.stack([int_to_u32(b, nl) for _, b in pairs]).view(np.int32)).cuda()
    C = torch.zeros((args.batch, npl), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    dp.mul_device(args.batch, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), npl, s)
    torch.cuda.synchronize()
    Cn = C.cpu().numpy().view(np.uint32)
    ok = all(u32_to_int(Cn[i]) == pairs[i][0] * pairs[i][1] for i in range(min(args.batch, 4)))
    ts = []
    for _ in range(args.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dp.mul_device(args.batch, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), npl, s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    prof = {}
    for _ in range(3):
        flush.zero_()
        for kind, ms, work, nbytes in dp.profile_device(args.batch, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), s):
            prof.setdefault(kind, []).append(ms)
    out[tw] = {"ms": round(ts[len(ts) // 2], 4), "exact": ok,
               "profile_ms": {k: round(sum(v) / 3, 4) for k, v in prof.items()}}
    dp.close()
out["speedup"] = round(out["cuda"]["ms"] / out["tensor"]["ms"], 3)
print(json.dumps(out))
