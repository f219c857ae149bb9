"""Randomised parity soak on the GPU: products of random sizes (and random word sizes / squares /
unbalanced operands) through dmul against Python's int product.

  python tools/soak.py [--n 200] [--max-bits 25] [--seed 1]
"""
import argparse
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1503_04955_b200 import dmul  # noqa: E402
from paper_1503_04955_b200.dkss import dmul_many  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200)
ap.add_argument("--max-bits", type=int, default=25)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--max-plans", type=int, default=0, help="override the plan caches' size (0: default)")
args = ap.parse_args()
if args.max_plans:
    import paper_1503_04955_b200.dkss as _D

    _D._MAX_PLANS = args.max_plans
r = random.Random(args.seed)
t0 = time.time()
bad = 0
for i in range(args.n):
    lb = r.uniform(10, args.max_bits)
    na = int(2 ** lb) + r.randrange(-7, 8)
    kind = r.randrange(6)
    nb = na if kind < 3 else max(1, int(na * r.uniform(0.01, 1.0)))
    a = r.getrandbits(na) | (1 << (na - 1))
    b = a if kind == 5 else r.getrandbits(nb) | 1
    if kind == 4:  # long carry chains
        a, b = (1 << na) - 1, (1 << nb) - 1
    got = dmul(a, b).to_int()
    if got != a * b:
        bad += 1
        x = got ^ (a * b)
        lo, hi = (x & -x).bit_length() - 1, x.bit_length()
        again = dmul(a, b).to_int() == a * b
        # which state is wrong: the device-resident path of the same device plan, a swapped call,
        # and a fresh device plan
        import numpy as np
        import torch
        import paper_1503_04955_b200.dkss as D
        from paper_1503_04955_b200.words import int_to_u32, u32_to_int

        plan, dp, nl, npl, _, _ = D._hot_plan(max(a.bit_length(), b.bit_length(), D._MIN_PLAN_BITS), 64)
        A = torch.from_numpy(int_to_u32(a, nl).view(np.int32)).cuda()
        B = torch.from_numpy(int_to_u32(b, nl).view(np.int32)).cuda()
        C = torch.zeros(npl, dtype=torch.int32, device="cuda")
        dp.mul_device(1, A.data_ptr(), B.data_ptr(), nl, C.data_ptr(), npl)
        torch.cuda.synchronize()
        dev_ok = u32_to_int(C.cpu().numpy().view(np.uint32)) == a * b
        swapped = dmul(b, a).to_int() == a * b
        small = dmul(a >> 1, b).to_int() == (a >> 1) * b
        D.clear_device_plans()
        fresh = dmul(a, b).to_int() == a * b
        print("MISMATCH", i, na, nb, kind, "plan", plan.M, plan.m, plan.u, "differing bits", lo, "..", hi, "of",
              (a * b).bit_length(), "popcount", bin(x).count("1"), "repeat ok:", again, "device-resident ok:", dev_ok,
              "swapped ok:", swapped, "a>>1 ok:", small, "fresh plan ok:", fresh, flush=True)
# a batch with ragged operand sizes
pairs = [(r.getrandbits(1 << 17) | 1, r.getrandbits(r.randrange(1, 1 << 17)) | 1) for _ in range(200)]
res = dmul_many(pairs)
bad += sum(1 for (a, b), c in zip(pairs, res) if c.to_int() != a * b)
print(f"soak: {args.n} products up to 2^{args.max_bits} bits + a ragged batch of 200, mismatches: {bad}, {time.time() - t0:.1f} s")
sys.exit(1 if bad else 0)
