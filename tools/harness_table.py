"""The thesis's run-time table through the REFERENCE's own harness: bigmul.bench.run_bench over
dmul and smul with both GPU rungs installed in the reference's ALGORITHMS table
(paper_1503_04955_b200.integration.install), the CSV of bigmul/bench.py:74-77 and the
T_DMUL / T_SMUL column of bigmul/bench.py:80-91.  Every timed product is checked by run_bench
against a "pyint" rung registered in the same table (Python's int product; the reference's
default t3mul rung is pure Python and takes minutes at 10^5 words).

  python tools/harness_table.py [--max-words 131072] [--csv out.csv]

Needs the reference package: baseline/_ref (pip --target install) or /root/reference/pkg/src.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(path, "bigmul")):
        sys.path.insert(0, path)
        break
sys.dont_write_bytecode = True

import bigmul  # noqa: E402
from bigmul.bench import FAVORABLE_WORDS, quotient_column, run_bench, write_csv  # noqa: E402
from bigmul.dispatch import ALGORITHMS  # noqa: E402
from bigmul.words import Natural  # noqa: E402

from paper_1503_04955_b200.integration import install  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-words", type=int, default=1 << 17)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--csv")
args = ap.parse_args()
sizes = sorted({1 << k for k in range(6, 18) if 1 << k <= args.max_words} |
               {s for s in FAVORABLE_WORDS if s <= args.max_words})
install(bigmul, smul=True)
ALGORITHMS["pyint"] = lambda a, b, table, arena: Natural.from_int(a.to_int() * b.to_int(), length=len(a) + len(b))
recs = run_bench(["dmul", "smul"], sizes, reps=args.reps, seed=1503, reference="pyint")
if args.csv:
    with open(args.csv, "w") as f:
        write_csv(recs, f)
        f.write("\n# input_words,T_DMUL/T_SMUL (end to end through the reference's run_bench)\n")
        for words, q in quotient_column(recs):
            f.write(f"# {words},{q:.3f}\n")
for words, q in quotient_column(recs):
    d = next(r.median_ns for r in recs if r.algorithm == "dmul" and r.input_words == words)
    s = next(r.median_ns for r in recs if r.algorithm == "smul" and r.input_words == words)
    print(f"{words:7d} words  dmul {d / 1e3:9.1f} us  smul {s / 1e3:9.1f} us  T_DMUL/T_SMUL {q:.3f}")
