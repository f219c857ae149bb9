"""Summaries of ncu output for profiles/.

  python tools/ncu_summary.py full <rep.ncu-rep> [--workload W] [--traffic profiles/ncu_traffic.json]
      per-kernel table of a `--set full` capture (device time, DRAM bytes, pipes, occupancy,
      top stall reasons); with --traffic, merges the per-launch DRAM bytes of each bench
      kernel kind into that JSON (bench.py reads it for roofline.traffic)
  python tools/ncu_summary.py launches <launches.csv>
      share of device time per kernel in a `--metrics gpu__time_duration.sum` launch list
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KIND = {"k_tc_twiddle": "twiddle_tc", "k_rows_dyn": "rows", "k_rows": "rows", "k_fwd_pass": "fwd_pass", "k_fwd_warp": "fwd_pass", "k_dft_cols": "fwd_pass", "k_inv_pass": "inv_pass",
        "k_inv_warp": "inv_pass", "k_bottom": "bottom", "k_decode1": "decode1", "k_decode2": "decode2",
        "k_decode_scan": "decode_scan", "k_encode": "encode"}


def _num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def kind_of(name):
    for k, v in KIND.items():
        if k in name:
            return v
    return name.split("(")[0][:40]


def full(rep, workload=None, traffic=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], dict(zip(r[0], r[1]))
    keys = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
            ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
            ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy%"),
            ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"), ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%")]
    scale = {"usecond": 1e3, "us": 1e3, "nsecond": 1.0, "ns": 1.0, "msecond": 1e6, "ms": 1e6, "byte": 1, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}
    per_kind = defaultdict(list)
    pipe = defaultdict(list)
    print(f"# {os.path.basename(rep)}" + (f" ({workload})" if workload else ""))
    print("kernel | " + " | ".join(k for _, k in keys) + " | top stalls")
    for row in r[2:]:
        d = dict(zip(hdr, row))
        name = d.get("Kernel Name", "")
        vals = []
        for k, short in keys:
            v = _num(d.get(k, ""))
            if v is not None and k in ("gpu__time_duration.sum",):
                v = v * scale.get(units.get(k, "nsecond"), 1.0)  # -> ns
            if v is not None and k.startswith("dram__bytes"):
                v = v * scale.get(units.get(k, "byte"), 1.0)  # -> bytes
            vals.append(v)
        st = [(_num(v), h) for h, v in d.items() if "smsp__pcsamp_warps_issue_stalled" in h and "not_issued" not in h
              and _num(v)]
        tot = sum(v for v, _ in st) or 1.0
        stalls = ", ".join(f"{h.split('stalled_')[1]} {100 * v / tot:.0f}%" for v, h in sorted(st, reverse=True)[:4])
        cells = []
        for (k, short), v in zip(keys, vals):
            if v is None:
                cells.append("-")
            elif short == "time":
                cells.append(f"{v / 1e3:.2f}us")
            elif short.startswith("dram"):
                cells.append(f"{v / 1e6:.3f}MB")
            else:
                cells.append(f"{v:.1f}" if v != int(v) else f"{int(v)}")
        print(f"{name.split('(')[0][:34]} | " + " | ".join(cells) + f" | {stalls}")
        if vals[1] is not None and vals[2] is not None:
            per_kind[kind_of(name)].append(vals[1] + vals[2])
        fh = vals[[k for _, k in keys].index("fmaheavy%")]
        if fh is not None:
            pipe[kind_of(name)].append(fh)
    if traffic and workload:
        data = {}
        if os.path.exists(traffic):
            with open(traffic) as f:
                data = json.load(f)
        w = data.setdefault(workload, {})
        for k, v in per_kind.items():
            w[k] = int(sum(v) / len(v))
        w["fmaheavy_pct"] = {k: round(sum(v) / len(v), 1) for k, v in pipe.items()}
        w["_source"] = (f"{os.path.basename(rep)}: dram__bytes_read.sum + dram__bytes_write.sum per launch (avg); "
                        "fmaheavy_pct = sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed (avg)")
        with open(traffic, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        print(f"# merged per-launch DRAM bytes into {traffic}: {dict((k, w[k]) for k in per_kind)}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    unit = data[0]["Metric Unit"] if data else "ns"
    mult = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6}.get(unit, 1.0)
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        n = d["Kernel Name"].split("(")[0].replace("void ", "")[:48]
        agg[n][0] += 1
        agg[n][1] += _num(d["Metric Value"]) * mult
    tot = sum(v[1] for v in agg.values())
    ours = sum(v[1] for n, v in agg.items() if "dkss" in n)
    print(f"# {os.path.basename(path)}: {len(data)} launches, {tot / 1e3:.1f} us device time "
          f"({ours / 1e3:.1f} us in libdkss kernels)")
    print("launches | total us | share of all | share of libdkss | avg us | kernel")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        sh = f"{100 * t / ours:5.1f}%" if "dkss" in n else "    -"
        print(f"{c:8d} | {t / 1e3:8.1f} | {100 * t / tot:5.1f}% | {sh} | {t / c / 1e3:7.2f} | {n}")


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    opts = dict(zip(sys.argv[3::2], sys.argv[4::2]))
    if mode == "full":
        full(path, opts.get("--workload"), opts.get("--traffic"))
    else:
        launches(path)
