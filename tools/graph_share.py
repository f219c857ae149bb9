"""Graph-replay device time of one multiply with phases skipped (DKSS_EXP_SKIP set by the
caller; products are wrong then): python tools/graph_share.py --bits 20"""
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
ap.add_argument("--steps", type=int, default=50)
args = ap.parse_args()
N = 1 << args.bits
r = random.Random(1)
dp = device_plan(_plan_for(N, 64))
nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
dA = torch.from_numpy(int_to_u32(r.getrandbits(N), nl).view(np.int32)).cuda()
dB = torch.from_numpy(int_to_u32(r.getrandbits(N), nl).view(np.int32)).cuda()
dC = torch.zeros(npl, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    dp.mul_device(1, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), npl, s.cuda_stream)
torch.cuda.synchronize()
tot = 0.0
for _ in range(args.steps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dp.mul_device(1, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), npl, s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
print(json.dumps({"skip": os.environ.get("DKSS_EXP_SKIP", "0"), "bits": args.bits, "us": round(1e3 * tot / args.steps, 2)}))
