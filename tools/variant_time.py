"""Device time of one multiply (or a batch) for every kernel-shape option of a plan
(include/dkss.h dkss_plan_opts), each checked against Python's int product.

  python tools/variant_time.py --bits 20 [--batch 1] [--reps 30]

Prints one JSON line per variant: graph-replay time (CUDA events, L2 flushed before every
replay) and the per-kind split from dkss_profile_device.
"""
import argparse
import itertools
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_04955_b200._native import DevicePlan  # noqa: E402
from paper_1503_04955_b200.dkss import _plan_for, plan_capacity  # noqa: E402
from paper_1503_04955_b200.words import int_to_u32, u32_to_int  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=20)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--twiddle", default="auto,cuda,tensor")
ap.add_argument("--pass-kind", default="auto")
ap.add_argument("--row-phase", default="auto")
args = ap.parse_args()

N = 1 << args.bits
r = random.Random(7)
plan = _plan_for(N, 64)
ai = [r.getrandbits(N) | 1 << (N - 1) for _ in range(args.batch)]
bi = [r.getrandbits(N) | 1 << (N - 1) for _ in range(args.batch)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
s = stream.cuda_stream

for tw, pk, rp in itertools.product(args.twiddle.split(","), args.pass_kind.split(","), args.row_phase.split(",")):
    try:
        dp = DevicePlan(plan_capacity(plan), plan.M, plan.m, plan.u, plan.p, plan.rho_powers, 0,
                        row_phase=rp, pass_kind=pk, twiddle=tw)
    except Exception as e:  # an option the plan does not support
        print(json.dumps({"twiddle": tw, "pass_kind": pk, "row_phase": rp, "error": str(e)}))
        continue
    nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
    dA = torch.from_numpy(np.stack([int_to_u32(x, nl) for x in ai]).view(np.int32)).cuda()
    dB = torch.from_numpy(np.stack([int_to_u32(x, nl) for x in bi]).view(np.int32)).cuda()
    dC = torch.zeros((args.batch, npl), dtype=torch.int32, device="cuda")
    dp.mul_device(args.batch, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), npl, s)
    torch.cuda.synchronize()
    C = dC.cpu().numpy().view(np.uint32)
    ok = all(u32_to_int(C[i]) == ai[i] * bi[i] for i in range(min(args.batch, 8)))
    times = []
    for rep in range(args.reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dp.mul_device(args.batch, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), npl, s)
        e1.record()
        torch.cuda.synchronize()
        if rep >= 3:
            times.append(e0.elapsed_time(e1))
    agg = {}
    for rep in range(4):
        flush.zero_()
        run = dp.profile_device(args.batch, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), s)
        if rep == 0:
            continue
        for kind, ms, work, nbytes in run:
            agg[kind] = agg.get(kind, 0.0) + ms / 3
    print(json.dumps({"bits": args.bits, "batch": args.batch, "twiddle": tw, "pass_kind": pk, "row_phase": rp,
                      "exact": ok, "median_us": round(1e3 * sorted(times)[len(times) // 2], 1),
                      "min_us": round(1e3 * min(times), 1), "launches": dp.info["launches_per_mul"],
                      **{k: round(v * 1e3, 1) for k, v in agg.items()}}), flush=True)
    dp.close()
