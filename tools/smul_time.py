"""Device time of one N x N-bit multiply by SMUL and by DKSS, and their quotient -- the
thesis's central measurement T_DMUL / T_SMUL (bigmul/bench.py:84-91
quotient_column).  CUDA events around stream-ordered device calls, operands resident in
HBM, L2 flushed before every timed call; the SMUL product is checked against a*b once.

  python tools/smul_time.py [--bits 16 18 20 22 24 26] [--reps 10] [--json out.json]
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
from paper_1503_04955_b200.smul import device_plan_for  # noqa: E402
from paper_1503_04955_b200.words import int_to_u32  # noqa: E402


def timed(fn, reps, flush):
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, nargs="+", default=[16, 18, 20, 22, 24, 26])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--json")
    args = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rows = []
    for e in args.bits:
        N = 1 << e
        r = random.Random(e)
        a, b = r.getrandbits(N) | 1 << (N - 1), r.getrandbits(N) | 1 << (N - 1)
        nl = N // 32
        dA = torch.from_numpy(int_to_u32(a, nl).view(np.int32)).cuda()
        dB = torch.from_numpy(int_to_u32(b, nl).view(np.int32)).cuda()
        sp, sdp = device_plan_for(2 * N, 64)
        dC = torch.zeros(sdp.product_limbs, dtype=torch.int32, device="cuda")
        run_s = lambda: sdp.mul_device(1, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), sdp.product_limbs, s)  # noqa
        run_s()
        torch.cuda.synchronize()
        ok = int.from_bytes(dC.cpu().numpy().view(np.uint32).tobytes(), "little") == a * b
        t_s = timed(run_s, args.reps, flush)
        dp = device_plan(_plan_for(N, 64))
        dnl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
        dA2 = torch.zeros(dnl, dtype=torch.int32, device="cuda")
        dB2 = torch.zeros(dnl, dtype=torch.int32, device="cuda")
        dA2[:nl] = dA
        dB2[:nl] = dB
        dC2 = torch.zeros(npl, dtype=torch.int32, device="cuda")
        run_d = lambda: dp.mul_device(1, dA2.data_ptr(), dB2.data_ptr(), dnl, dC2.data_ptr(), npl, s)  # noqa
        t_d = timed(run_d, args.reps, flush)
        row = {"bits": e, "smul_ms": round(t_s, 4), "dmul_ms": round(t_d, 4), "dmul_over_smul": round(t_d / t_s, 2),
               "smul_plan": {"m": sp.m, "K": sp.K, "s": sp.s}, "smul_gbit_s": round(2 * N / t_s / 1e6, 2),
               "smul_exact": ok}
        print(json.dumps(row), flush=True)
        rows.append(row)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
