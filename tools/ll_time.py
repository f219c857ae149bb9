"""Time the device Lucas-Lehmer loop: python tools/ll_time.py 21701 44497 86243"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1503_04955_b200.lucas import lucas_lehmer, lucas_lehmer_steps  # noqa: E402

for p in map(int, sys.argv[1:] or ["21701"]):
    lucas_lehmer_steps(p, 20, 4)  # plan upload + graph capture
    t0 = time.perf_counter()
    verdict, res = lucas_lehmer(p, "dmul")
    dt = time.perf_counter() - t0
    print(json.dumps({"p": p, "is_prime": verdict, "residue64": f"0x{res:016x}", "seconds": round(dt, 3),
                      "us_per_iteration": round(1e6 * dt / (p - 2), 2)}), flush=True)
