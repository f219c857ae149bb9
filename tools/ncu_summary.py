"""Summaries of an ncu report: python tools/ncu_summary.py <rep> [--source]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
for row in r[2:]:
    d = dict(zip(hdr, row))
    print("kernel:", d.get("Kernel Name", "")[:90], "| duration", d.get("gpu__time_duration.sum"), "ns")
    keys = ["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
    for k in keys:
        if k in d:
            print(f"   {k:70s} {d[k]}")
    st = [(float(v), h) for h, v in d.items() if "smsp__pcsamp_warps_issue_stalled" in h and "not_issued" not in h
          and v.replace('.', '', 1).isdigit() and float(v) > 0]
    tot = sum(v for v, _ in st)
    print("   stalls:", ", ".join(f"{h.split('stalled_')[1]} {100 * v / tot:.0f}%" for v, h in sorted(st, reverse=True)[:8]))
if "--source" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    data = [dict(zip(hdr, x)) for x in rows[2:]]
    S, X = "Warp Stall Sampling (All Samples)", "Instructions Executed"
    tot = sum(float(d[S] or 0) for d in data)
    totx = sum(float(d[X] or 0) for d in data)
    blk = 64
    for i in range(0, len(data), blk):
        seg = data[i:i + blk]
        s = sum(float(d[S] or 0) for d in seg)
        x = sum(float(d[X] or 0) for d in seg)
        ops = {}
        for d in seg:
            t = d["Source"].split()
            if not t:
                continue
            o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[o] = ops.get(o, 0) + float(d[X] or 0)
        top = sorted(ops.items(), key=lambda kv: -kv[1])[:4]
        if s / tot > 0.005:
            print(f"{i:5d} samp {100 * s / tot:5.1f}% inst {100 * x / totx:5.1f}%  {[(k, round(100 * v / totx, 1)) for k, v in top]}")
