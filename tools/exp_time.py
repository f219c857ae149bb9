"""Per-kernel-kind device time of one multiply (no correctness check; for experiment builds).

  DKSS_LIB=paper_1503_04955_b200/_lib/libdkss_<variant>.so python tools/exp_time.py --bits 20 [--batch 1]
"""
import argparse
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_04955_b200.dkss import _plan_for, device_plan  # noqa: E402
from paper_1503_04955_b200.words import int_to_u32  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=20)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--reps", type=int, default=6)
args = ap.parse_args()
N = 1 << args.bits
r = random.Random(1)
plan = _plan_for(N, 64)
dp = device_plan(plan)
nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
A = np.stack([int_to_u32(r.getrandbits(N), nl) for _ in range(args.batch)])
B = np.stack([int_to_u32(r.getrandbits(N), nl) for _ in range(args.batch)])
dA = torch.from_numpy(A.view(np.int32)).cuda()
dB = torch.from_numpy(B.view(np.int32)).cuda()
dC = torch.zeros((args.batch, npl), dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
agg = {}
for rep in range(args.reps):
    flush.zero_()
    run = dp.profile_device(args.batch, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), s)
    if rep == 0:
        continue
    for kind, ms, work, nbytes in run:
        agg[kind] = agg.get(kind, 0.0) + ms / (args.reps - 1)
lib = os.path.basename(os.environ.get("DKSS_LIB", "libdkss.so"))
print(json.dumps({"lib": lib, "bits": args.bits, "batch": args.batch, **{k: round(v * 1e3, 1) for k, v in agg.items()},
                  "total_us": round(sum(agg.values()) * 1e3, 1)}))
