"""Decode SASS control bits (stall/yield/barriers/reuse) for a kernel: python tools/sass_ctrl.py <bin> <name-substr> [start] [count]"""
import re
import subprocess
import sys

binary, pat = sys.argv[1], sys.argv[2]
start = int(sys.argv[3]) if len(sys.argv) > 3 else 0
count = int(sys.argv[4]) if len(sys.argv) > 4 else 80
sass = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    if pat not in dem:
        continue
    lines = f.split("\n")
    ins = []
    for i, l in enumerate(lines):
        m = re.match(r"\s+/\*([0-9a-f]{4})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", l)
        if m and i + 1 < len(lines):
            m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
            hi = int(m2.group(1), 16) if m2 else 0
            ins.append((m.group(1), m.group(2), hi))
    print(dem[:100], len(ins), "instructions")
    hist = {}
    for addr, txt, hi in ins:
        op = txt.split()[0] if not txt.startswith("@") else txt.split()[1]
        st = (hi >> 41) & 0xF
        hist.setdefault(op, {}).setdefault(st, 0)
        hist[op][st] += 1
    for op in ("IMAD.WIDE.U32", "IMAD.WIDE", "IMAD.MOV.U32", "LOP3.LUT", "LDS", "IADD3"):
        if op in hist:
            print("  stall histogram", op, dict(sorted(hist[op].items())))
    for addr, txt, hi in ins[start:start + count]:
        st, y, wb, rb, wm, ru = (hi >> 41) & 0xF, (hi >> 45) & 1, (hi >> 46) & 7, (hi >> 49) & 7, (hi >> 52) & 0x3F, (hi >> 58) & 0xF
        print(f"  {addr} S{st:02d} Y{y} wb{wb} rb{rb} wt{wm:02x} ru{ru:x}  {txt[:70]}")
    break
