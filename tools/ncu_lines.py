"""Stall samples per CUDA source line of one kernel in an ncu report (needs -lineinfo).
  python tools/ncu_lines.py <rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kre}",
                      "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname = [], None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        x = float(d.get("Instructions Executed", 0) or 0)
        res.append((s, x, fname, int(r[0]), r[1].strip()[:70]))
tot = sum(r[0] for r in res) or 1
totx = sum(r[1] for r in res) or 1
for s, x, f, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% samp {100 * x / totx:5.1f}% inst  {f}:{ln}  {src}")
