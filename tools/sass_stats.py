"""Opcode histogram of one kernel in a cubin/so/exe: python tools/sass_stats.py <binary> <name-substring>"""
import re
import subprocess
import sys

binary, pat = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    if pat not in dem:
        continue
    ops = re.findall(r"^\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", f, re.M)
    hist = {}
    for o in ops:
        hist[o] = hist.get(o, 0) + 1
    top = sorted(hist.items(), key=lambda kv: -kv[1])[:12]
    print(dem[:110])
    print("   total", len(ops), " ".join(f"{k}:{v}" for k, v in top))
