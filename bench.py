"""Benchmark: N x N-bit DKSS multiply on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config mul2^20|ones2^20|batch1024x2^18|mul2^24|mul2^26|mul2^16]

One JSON line on rank 0.  A "step" is one pass of the hot path over one batch
of synthetic input: for the default workload (BASELINE.json configs[1],
2^20 x 2^20 bits, uniform random with the top bit set) one full DKSS
multiply.  `value` = product Gbit/s (2N bits per product / device time), whole
job over all ranks.  Multi-GPU runs are weak-scaled independent multiplies (one
per rank per step, no data-path collective) unless `--split` is given: then ONE
multiply per step is split over the ranks with the four-step layout (SURVEY.md
§8(e); NCCL all-to-all between the column and row phases, strong scaling).

Timing: CUDA events on the launching stream around every step, an L2 flush
(256 MiB memset, outside the events) before every timed step, barrier +
synchronize around the whole timed region, max over ranks.  SM clocks and
throttle reasons are sampled with NVML during the timed region.

`--impl reference` times the reference algorithm's CPU path: the C port of
bigmul/dkss.py in oracle/ (the reference itself is pure Python and cannot be
installed on the GPU box), on all host threads, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

CONFIGS = {
    # name: (N bits, batch, seed, all_ones)
    "mul2^16": (1 << 16, 1, 1, False),
    "mul2^20": (1 << 20, 1, 2, False),
    "ones2^20": (1 << 20, 1, 0, True),
    "batch1024x2^18": (1 << 18, 1024, 3, False),
    "mul2^24": (1 << 24, 1, 4, False),
    "mul2^26": (1 << 26, 1, 5, False),
}
DEFAULT_CONFIG = "mul2^20"


def operands(N: int, batch: int, seed: int, ones: bool, rank: int = 0):
    """Seeded operands, generated as random.Random(seed).getrandbits(N) | 1<<(N-1);
    batch pair i uses seed + i; ranks > 0 offset the seed by 1_000_003 * rank."""
    out = []
    for i in range(batch):
        if ones:
            a = b = (1 << N) - 1
        else:
            r = random.Random(seed + i + 1_000_003 * rank)
            a = r.getrandbits(N) | 1 << (N - 1)
            b = r.getrandbits(N) | 1 << (N - 1)
        out.append((a, b))
    return out


def imad_peak():
    """Measured IMAD.WIDE.U32 issue rate (32x32->64 products/s) from profiles/imad_peak.json."""
    path = os.path.join(HERE, "profiles", "imad_peak.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["peak_products_per_s"]), d.get("source", "profiles/imad_peak.json")
    # SURVEY.md §8(d) planning assumption (64 IMAD/clk/SM x 148 x 1.965 GHz / 2)
    return 9.3e12, "fallback: SURVEY.md planning assumption"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device: int, period_s: float = 0.002):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.max_mhz = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:  # noqa: BLE001
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for bit, name in self.REASONS.items():
            if r & bit and bit != 0x1:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()
            self._sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def cpu_baseline(N, pairs, budget_s: float, threads: int | None = None):
    """Time the oracle (C port of bigmul/dkss.py) on host cores for ~budget_s."""
    from oracle.oracle import OraclePlan, max_threads, set_threads
    from paper_1503_04955_b200.plan import dkss_select_params

    threads = threads or os.cpu_count() or 1
    set_threads(threads)
    plan = dkss_select_params(N)
    op = OraclePlan(plan)
    done, t0 = 0, time.perf_counter()
    a, b = pairs[0]
    c = op.dmul(a, b)
    if c != a * b:
        raise SystemExit("oracle mismatch")
    done = 1
    while time.perf_counter() - t0 < budget_s and done < 1000:
        a, b = pairs[done % len(pairs)]
        op.dmul(a, b)
        done += 1
    dt = time.perf_counter() - t0
    return {"value": 2 * N * done / dt / 1e9, "unit": "Gbit/s", "cores": min(threads, max_threads()),
            "kind": "port", "sample": f"{done} x 2^{N.bit_length() - 1}-bit dmul by oracle/dkss_oracle.c "
                                      f"({threads} OpenMP threads, {dt:.1f}s)",
            "ms_per_mul": 1e3 * dt / done}


def run_reference(args, cfg_name):
    N, batch, seed, ones = CONFIGS[cfg_name]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pairs = operands(N, min(batch, 8), seed, ones)
    from oracle.oracle import OraclePlan, set_threads
    from paper_1503_04955_b200.plan import dkss_select_params
    threads = os.cpu_count() or 1
    set_threads(threads)
    op = OraclePlan(dkss_select_params(N))
    a, b = pairs[0]
    assert op.dmul(a, b) == a * b
    for i in range(args.warmup):
        op.dmul(*pairs[i % len(pairs)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        op.dmul(*pairs[i % len(pairs)])
    dt = time.perf_counter() - t0
    # a step of the batched config is `batch` products; the oracle runs a bounded sample
    value = 2 * N * args.steps / dt / 1e9
    line = {"metric": "N x N-bit DKSS multiply: product Gbit/s", "value": round(value, 6), "unit": "Gbit/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (seeded random operands)",
            "config": {"workload": cfg_name, "bits": N, "batch": 1,
                       "note": "each step = one product by the C port of bigmul/dkss.py (bounded sample)"},
            "cpu_baseline": {"value": round(value, 6), "unit": "Gbit/s", "cores": threads, "kind": "port",
                             "sample": f"{args.steps} x 2^{N.bit_length() - 1}-bit products, {dt:.2f}s"},
            "e2e": {"value": round(value, 6), "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_split(args):
    """One multiply per step, split over all ranks (four-step, NCCL all-to-all)."""
    import torch
    import torch.distributed as dist

    from paper_1503_04955_b200.dkss import set_device
    from paper_1503_04955_b200.fourstep import DistExchange, _operands, dmul_fourstep, make_rank, run_rank
    from paper_1503_04955_b200.plan import dkss_select_params, ring_products_per_multiply

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world < 2:
        raise SystemExit("--split needs torchrun with >= 2 ranks (tests emulate ranks on one GPU)")
    gloo = os.environ.get("DKSS_BENCH_GLOO", "0") not in ("", "0")  # see main()
    if gloo:
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if gloo:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    os.environ["DKSS_DEVICE"] = str(local)
    set_device(local)
    N, batch, seed, ones = CONFIGS[args.config]
    if batch != 1:
        raise SystemExit("--split applies to single-multiply configs")
    a, b = operands(N, 1, seed, ones, 0)[0]  # every rank holds the same operands
    plan = dkss_select_params(N)
    fs = make_rank(plan, rank, world, dev)
    A, B = _operands(plan, a, b, dev)
    ex = DistExchange()
    stream = torch.cuda.current_stream(dev)
    prod = run_rank(fs, ex, A, B)
    torch.cuda.synchronize(dev)
    if rank == 0 and int.from_bytes(prod.cpu().numpy().view("uint32").tobytes(), "little") != a * b:
        raise SystemExit("split product mismatch")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        flush.zero_()
        run_rank(fs, ex, A, B)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize(dev)
    with clocks:
        for k in range(args.steps):
            flush.zero_()
            dist.barrier()
            starts[k].record(stream)
            run_rank(fs, ex, A, B)
            ends[k].record(stream)
        torch.cuda.synchronize(dev)
    dist.barrier()
    t = torch.tensor([sum(s.elapsed_time(e) for s, e in zip(starts, ends))], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    e2e = []
    for _ in range(3):
        dist.barrier()
        t0 = time.perf_counter()
        dmul_fourstep(a, b)
        e2e.append(time.perf_counter() - t0)
    e2e_s = sorted(e2e)[1]
    if rank == 0:
        peak, peak_src = imad_peak()
        info = fs.stages.dp.info
        w_mul = ring_products_per_multiply(plan) * plan.m * plan.m * info["L"] * info["L"]
        per_gpu = w_mul / world / (ms_per_step * 1e-3)
        lay = fs.stages.layout(world)
        line = {
            "metric": "N x N-bit DKSS multiply: product Gbit/s", "value": round(2 * N / (ms_per_step * 1e-3) / 1e9, 4),
            "unit": "Gbit/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 5), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (seeded random operands, SURVEY.md §8(d))",
            "config": {"workload": args.config, "bits": N, "batch": 1, "parallelism": f"four-step split x{world}",
                       "exchange_bytes_per_rank": 3 * 4 * lay["block_words"] * (world - 1) // world,
                       "l2": "flushed (256 MiB memset) before every timed step"},
            "roofline": {"bound": "imad", "achieved": round(per_gpu / 1e12, 4), "peak": round(peak / 1e12, 4),
                         "unit": "T limb-products/s per GPU", "frac": round(per_gpu / peak, 4), "traffic": None,
                         "kernel": "whole split multiply", "peak_source": peak_src},
            "e2e": {"value": round(2 * N / e2e_s / 1e9, 4), "unit": "Gbit/s", "ms": round(e2e_s * 1e3, 3),
                    "h2d_bytes_per_step": 2 * A.numel() * 4 * world, "d2h_bytes_per_step": fs.prod.numel() * 4,
                    "api": "paper_1503_04955_b200.fourstep.dmul_fourstep(int, int)"},
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--split", action="store_true", help="four-step split of one multiply over the ranks")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args, args.config)
        return
    if args.split:
        run_split(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DKSS_BENCH_GLOO=1: run the multi-rank path with gloo and ranks sharing the visible GPUs
    # (checks the orchestration on a 1-GPU box; NCCL needs one GPU per rank)
    gloo = os.environ.get("DKSS_BENCH_GLOO", "0") not in ("", "0")
    if gloo:
        local %= max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    os.environ["DKSS_DEVICE"] = str(local)

    from paper_1503_04955_b200.dkss import device_plan, dmul, dmul_many, set_device
    set_device(local)
    from paper_1503_04955_b200.plan import dkss_select_params, ring_products_per_multiply
    from paper_1503_04955_b200.words import int_to_u32, u32_to_int

    N, batch, seed, ones = CONFIGS[args.config]
    pairs = operands(N, batch, seed, ones, rank)
    plan = dkss_select_params(N)
    dp = device_plan(plan, local)
    info = dp.info
    nl, npl = info["operand_limbs"], info["product_limbs"]
    A = np.stack([int_to_u32(a, nl) for a, _ in pairs])
    B = np.stack([int_to_u32(b, nl) for _, b in pairs])
    dA = torch.from_numpy(A.view(np.int32)).to(dev)
    dB = torch.from_numpy(B.view(np.int32)).to(dev)
    dC = torch.zeros((batch, npl), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def step():
        dp.mul_device(batch, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), npl, sp)

    # correctness gate (bigmul/bench.py:66-68 style): every product bit-exact vs Python ints
    step()
    torch.cuda.synchronize(dev)
    C = dC.cpu().numpy().view(np.uint32)
    check = range(batch) if batch <= 64 else list(range(0, batch, max(1, batch // 64)))
    for i in check:
        a, b = pairs[i]
        if u32_to_int(C[i]) != a * b:
            raise SystemExit(f"product mismatch at pair {i}")

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with clocks:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            starts[k].record(stream)
            step()
            ends[k].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    ms_per_step = max_ms / args.steps
    products = batch * world * args.steps
    value = 2 * N * products / (max_ms * 1e-3) / 1e9

    # per-launch profile (CUDA events between the same launches, un-graphed)
    prof_runs = []
    for _ in range(5):
        flush.zero_()
        prof_runs.append(dp.profile_device(batch, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), sp))
    per_kind = {}
    for run in prof_runs[1:]:
        for kind, ms, work, nbytes in run:
            d = per_kind.setdefault(kind, {"ms": 0.0, "work": 0, "bytes": 0, "launches": 0})
            d["ms"] += ms
            d["work"] += work
            d["bytes"] += nbytes
            d["launches"] += 1
    nprof = len(prof_runs) - 1
    for d in per_kind.values():
        d["ms_per_mul"] = d["ms"] / nprof
    launches = len(prof_runs[0])
    dom = max(per_kind, key=lambda k: per_kind[k]["ms"])
    dk = per_kind[dom]
    peak, peak_src = imad_peak()
    achieved = dk["work"] / (dk["ms"] * 1e-3) if dk["ms"] > 0 else 0.0
    rp = ring_products_per_multiply(plan)
    w_mul = rp * plan.m * plan.m * info["L"] * info["L"]
    prof_total_ms = sum(d["ms_per_mul"] for d in per_kind.values())
    traffic, pipe_pct = None, None
    tpath = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            nt = json.load(f).get(args.config, {})
        traffic = nt.get(dom)
        pipe_pct = nt.get("fmaheavy_pct", {}).get(dom)

    # end to end through the public API (Python ints in, Natural / ints out; H2D + D2H inside):
    # dmul for one product, dmul_many for the batched workload (one device call per step)
    e2e_times = []
    a0, b0 = pairs[0]
    if batch == 1:
        def e2e_call():
            return [dmul(a0, b0)]  # -> Natural, as the reference's dmul returns
    else:
        def e2e_call():
            return dmul_many(pairs)
    e2e_call()
    for _ in range(max(3, args.e2e_steps if batch == 1 else args.e2e_steps // 4)):
        t0 = time.perf_counter()
        r = e2e_call()
        e2e_times.append(time.perf_counter() - t0)
    if r[0].to_int() != a0 * b0 or r[-1].to_int() != pairs[len(r) - 1][0] * pairs[len(r) - 1][1]:
        raise SystemExit("e2e product mismatch")
    e2e_times.sort()
    e2e_s = e2e_times[len(e2e_times) // 2]

    # the thesis's comparison baseline on the same operands: SMUL device time and T_DMUL / T_SMUL
    # (bigmul/bench.py:80-91), L2 flushed before every call
    smul_line = None
    try:
        from paper_1503_04955_b200.smul import device_plan_for
        splan, sdp = device_plan_for(2 * N, 64)
        snc = sdp.product_limbs
        dS = torch.zeros((batch, snc), dtype=torch.int32, device=dev)

        def sstep():
            sdp.mul_device(batch, dA.data_ptr(), dB.data_ptr(), nl, dS.data_ptr(), snc, sp)

        sstep()
        torch.cuda.synchronize(dev)
        S0 = dS[0].cpu().numpy().view(np.uint32)
        sts = []
        for i in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sstep()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if i >= 2:
                sts.append(e0.elapsed_time(e1))
        s_ms = float(np.median(sts))
        smul_line = {"ms_per_step": round(s_ms, 5), "gbit_s": round(2 * N * batch / (s_ms * 1e-3) / 1e9, 4),
                     "dmul_over_smul": round(ms_per_step / s_ms, 3), "exact": u32_to_int(S0) == pairs[0][0] * pairs[0][1],
                     "plan": {"m": splan.m, "K": splan.K, "s": splan.s}}
    except Exception as e:  # the headline does not depend on it; say why it is missing
        smul_line = {"unavailable": repr(e)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(N, pairs[:4], args.cpu_budget)

    if rank == 0:
        line = {
            "metric": "N x N-bit DKSS multiply: product Gbit/s", "value": round(value, 4), "unit": "Gbit/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded random operands, SURVEY.md §8(d))",
            "config": {"workload": args.config, "bits": N, "batch_per_rank": batch, "plan": {
                "M": plan.M, "m": plan.m, "u": plan.u, "d": plan.d, "levels": plan.levels, "base": plan.base_len},
                "l2": "flushed (256 MiB memset) before every timed step", "parallelism": f"replicas x{world}"},
            "roofline": {"bound": "imad", "achieved": round(achieved / 1e12, 4), "peak": round(peak / 1e12, 4),
                         "unit": "T limb-products/s (32x32->64)", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "kernel": dom, "peak_source": peak_src,
                         "ncu_fmaheavy_pct": pipe_pct,  # IMAD.WIDE pipe busy, from the committed ncu capture
                         "work_per_launch": dk["work"] // max(1, dk["launches"]),
                         "whole_multiply_frac": round(w_mul / (ms_per_step * 1e-3 / batch) / peak, 4) if batch == 1
                         else round(w_mul * batch / (ms_per_step * 1e-3) / peak, 4)},
            "kernels": {k: {"ms_per_mul": round(v["ms_per_mul"], 5), "launches_per_mul": v["launches"] // nprof,
                            "work": v["work"] // nprof,
                            "tput_T_per_s": round(v["work"] / (v["ms"] * 1e-3) / 1e12, 3) if v["work"] else 0}
                        for k, v in per_kind.items()},
            "profile_total_ms": round(prof_total_ms, 5),
            "ring_products_per_mul": rp, "w_mul_limb_products": w_mul,
            "gpu_launches": launches * args.steps,  # libdkss kernels in the timed region (flush memset excluded)
            "gpu_launches_per_step": launches,
            "e2e": {"value": round(2 * N * batch * world / e2e_s / 1e9, 4), "unit": "Gbit/s",
                    "ms": round(e2e_s * 1e3, 4),
                    "h2d_bytes_per_step": 2 * nl * 4 * batch, "d2h_bytes_per_step": npl * 4 * batch,
                    "api": "paper_1503_04955_b200.dmul(int, int) -> Natural" if batch == 1 else
                           "paper_1503_04955_b200.dmul_many([(int, int)] * batch) -> [Natural]"},
            "clocks": clocks.summary(),
            "smul": smul_line,
        }
        if cpu:
            line["cpu_baseline"] = {k: v for k, v in cpu.items() if k != "ms_per_mul"}
            line["cpu_baseline"]["value"] = round(line["cpu_baseline"]["value"], 6)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
