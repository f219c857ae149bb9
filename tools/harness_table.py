"""The thesis's run-time table through the reference-style harness: run_bench over dmul and
smul (both on the GPU, every timed product checked against Python's int product), the CSV
of bigmul/bench.py:74-77 and the T_DMUL / T_SMUL column of bigmul/bench.py:80-91.

  python tools/harness_table.py [--max-words 131072] [--csv out.csv]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1503_04955_b200.harness import FAVORABLE_WORDS, quotient_column, run_bench, write_csv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-words", type=int, default=1 << 17)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--csv")
args = ap.parse_args()
sizes = sorted({1 << k for k in range(6, 18) if 1 << k <= args.max_words} |
               {s for s in FAVORABLE_WORDS if s <= args.max_words})
recs = run_bench(["dmul", "smul"], sizes, reps=args.reps, seed=1503)
if args.csv:
    with open(args.csv, "w") as f:
        write_csv(recs, f)
        f.write("\n# input_words,T_DMUL/T_SMUL (end to end through ALGORITHMS, host ints in)\n")
        for words, q in quotient_column(recs):
            f.write(f"# {words},{q:.3f}\n")
for words, q in quotient_column(recs):
    d = next(r.median_ns for r in recs if r.algorithm == "dmul" and r.input_words == words)
    s = next(r.median_ns for r in recs if r.algorithm == "smul" and r.input_words == words)
    print(f"{words:7d} words  dmul {d / 1e3:9.1f} us  smul {s / 1e3:9.1f} us  T_DMUL/T_SMUL {q:.3f}")
