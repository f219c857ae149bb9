"""Benchmark: N x N-bit DKSS multiply on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config mul2^24|mul2^20|ones2^20|batch1024x2^18|mul2^26|mul2^16] [--replicas]

One JSON line on rank 0.  A "step" is one pass of the hot path over one batch of
synthetic input.  The default workload is BASELINE.json configs[3], the largest
single-GPU config: ONE 2^24 x 2^24-bit multiply, uniform random bits with the top bit
set (seed 4).  `value` = product Gbit/s (2N bits per product / device time), whole job.

Multi-GPU (`--gpus N`; without torchrun the script re-launches itself under
`torch.distributed.run`, one rank per GPU):
  * single-multiply configs: the multiply is split four-step over the ranks (SURVEY.md
    §8(e), fourstep.py: column phase, NCCL all-to-all, row phase, all-to-all back), strong
    scaling; `--replicas` runs independent copies instead (weak scaling);
  * batch1024x2^18: the fixed 1024 pairs are sharded by pair (parallel.shard_range), no
    data-path collective, strong scaling.
DKSS_BENCH_GLOO=1 runs the ranks over gloo with every rank on the visible GPU(s): it checks
the orchestration on a one-GPU box (NCCL needs one GPU per rank).

Correctness gate before any timing (bigmul/bench.py:57-68 checks every product): every
product of the first step is checked -- single products against Python's `a*b` (2^26:
residues modulo 64 seeded 62-bit primes, as BASELINE.json config 5 allows), the batch by
residues for every pair plus the full product for a sample.

Timing: CUDA events on the launching stream around every step, an L2 flush (256 MiB
memset, outside the events) before every timed step, barrier + synchronize around the
timed region, max over ranks.  SM clocks and throttle reasons are sampled with NVML
during the timed region.  `gpu_launches` is the libdkss kernel count inside the timed
region (dkss_kernel_launches(); graph replays count their kernel nodes).

`--impl reference` times the reference algorithm's CPU path on the host cores: the C
restatement of bigmul/dkss.py in oracle/ (the reference itself is pure Python; it cannot be
shipped to the GPU box and would measure the interpreter, 41 s per 2^20 multiply, BASELINE.md
§2), all host threads, rank 0 only, a bounded sample per step.  Both arms print the same
`config` dict.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import socket
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

CONFIGS = {
    # name: (N bits, pairs, seed, all_ones) -- BASELINE.json configs / SURVEY.md §8(d)
    "mul2^16": (1 << 16, 1, 1, False),
    "mul2^20": (1 << 20, 1, 2, False),
    "ones2^20": (1 << 20, 1, 0, True),
    "batch1024x2^18": (1 << 18, 1024, 3, False),
    "mul2^24": (1 << 24, 1, 4, False),
    "mul2^26": (1 << 26, 1, 5, False),
}
DEFAULT_CONFIG = "mul2^24"
METRIC = "N x N-bit DKSS multiply: product Gbit/s"
L2_NOTE = "flushed (256 MiB memset) before every timed GPU step"
FULL_CHECK_MAX_BITS = 1 << 24  # above this the gate uses residues (Python a*b at 2^26 takes ~90 s)


def operand_pair(N: int, seed: int, i: int, ones: bool):
    """Pair i of a config: random.Random(seed + i).getrandbits(N) | 1 << (N-1) for a, then b
    (SURVEY.md §8(d)); the all-ones pair is (2^N - 1, 2^N - 1)."""
    if ones:
        return (1 << N) - 1, (1 << N) - 1
    r = random.Random(seed + i)
    a = r.getrandbits(N) | 1 << (N - 1)
    b = r.getrandbits(N) | 1 << (N - 1)
    return a, b


def mode_for(cfg: str, world: int, replicas: bool) -> str:
    if CONFIGS[cfg][1] > 1:
        return "shard"
    if world == 1:
        return "single"
    return "replicas" if replicas else "split"


def config_dict(cfg: str, world: int, mode: str) -> dict:
    """The workload description both arms print (identical for the same arguments)."""
    N, pairs, seed, ones = CONFIGS[cfg]
    par = {
        "single": "1 GPU",
        "split": f"four-step split of each multiply over {world} GPUs",
        "shard": f"{pairs} pairs sharded by pair over {world} GPU(s), no data-path collective",
        "replicas": f"{world} independent replicas (one multiply per GPU per step)",
    }[mode]
    return {"workload": cfg, "bits": N, "pairs_per_step": pairs * (world if mode == "replicas" else 1),
            "operands": "all ones (2^N - 1)" if ones else f"Random(seed + i).getrandbits(N) | 1 << (N-1), seed {seed}",
            "parallelism": par, "n_gpus": world, "l2": L2_NOTE}


def scaling_for(mode: str) -> str:
    return "weak" if mode == "replicas" else "strong"


def check_primes(k: int, seed: int = 777):
    """k seeded random 62-bit primes (Miller-Rabin with fixed bases: deterministic below 2^64)."""
    pr = random.Random(seed)
    out = []
    while len(out) < k:
        q = pr.getrandbits(62) | 1 << 61 | 1
        d, s = q - 1, 0
        while d % 2 == 0:
            d //= 2
            s += 1
        ok = True
        for w in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
            x = pow(w, d, q)
            if x in (1, q - 1):
                continue
            for _ in range(s - 1):
                x = x * x % q
                if x == q - 1:
                    break
            else:
                ok = False
                break
        if ok:
            out.append(q)
    return out


def residues_ok(c: int, a: int, b: int, primes) -> bool:
    return all(c % q == (a % q) * (b % q) % q for q in primes)


def imad_peak():
    """Measured IMAD.WIDE.U32 issue rate (32x32->64 products/s) from profiles/imad_peak.json."""
    path = os.path.join(HERE, "profiles", "imad_peak.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["peak_products_per_s"]), d.get("source", "profiles/imad_peak.json")
    # SURVEY.md §8(d) planning assumption (64 IMAD/clk/SM x 148 x 1.965 GHz / 2)
    return 9.3e12, "fallback: SURVEY.md planning assumption"


def tc_i8_peak():
    """Measured dense int8 tensor-core rate (ops/s) from profiles/tc_i8_peak.json
    (tools/microbench_tc_i8.cu: tcgen05.mma kind::i8 M128 N256 K32 back to back on every SM)."""
    path = os.path.join(HERE, "profiles", "tc_i8_peak.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["ops_per_s"]), "tools/microbench_tc_i8.cu (profiles/tc_i8_peak.json)"
    return 4.5e15, "fallback: nominal dense int8 (2x the 2.25 PFLOP/s bf16 figure)"


def hbm_peak():
    """HBM bytes/s: MEASURED_PEAKS.json (driver-written), else the profiling recipe's fallback."""
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]) * 1e9, "MEASURED_PEAKS.json hbm_gbs"
    return 6.65e12, "fallback 6.65 TB/s (B200_PROFILING.md)"


# which roofline bounds each profiled kernel kind (bench's per-launch profile, dkss_profile_device)
TENSOR_KINDS = {"twiddle_tc"}                            # work = int8 ops of the byte GEMM
IMAD_KINDS = {"fwd_pass", "inv_pass", "bottom", "rows"}  # work = 32x32->64 limb products


def kernel_roofline(kind: str, work: int, nbytes: int, ms: float, peaks) -> dict:
    """Roofline of one kernel kind over a step: the slower of its compute at the matching peak and
    its stage bytes at HBM bandwidth; achieved / peak in the binding unit."""
    (imad, _), (tc, _), (hbm, _) = peaks
    s = ms * 1e-3
    if kind in TENSOR_KINDS:
        t_c, cu, cpk = work / tc, "T int8 ops/s", tc
    elif kind in IMAD_KINDS and work:
        t_c, cu, cpk = work / imad, "T limb-products/s (32x32->64)", imad
    else:
        t_c, cu, cpk = 0.0, None, None
    t_m = nbytes / hbm
    if t_c >= t_m and cu:
        bound, achieved, peak, unit = ("tensor" if kind in TENSOR_KINDS else "imad"), work / s, cpk, cu
    else:
        bound, achieved, peak, unit = "hbm", nbytes / s, hbm, "GB/s"
    scale = 1e9 if unit == "GB/s" else 1e12
    return {"bound": bound, "achieved": round(achieved / scale, 4), "peak": round(peak / scale, 4), "unit": unit,
            "frac": round(achieved / peak, 4), "t_roof_ms": round(max(t_c, t_m) * 1e3, 5)}


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


# ---------------------------------------------------------------------------
# the reference arm and the CPU baseline (oracle: C restatement of bigmul/dkss.py)

def _oracle_sample(N: int, pairs, threads: int):
    """One bounded sample: the pairs multiplied by the oracle on `threads` host threads."""
    import numpy as np

    from oracle.oracle import OraclePlan, set_threads
    from paper_1503_04955_b200.plan import dkss_select_params

    set_threads(threads)
    op = OraclePlan(dkss_select_params(N))
    nl = -(-N // 32)
    A = np.stack([np.frombuffer(a.to_bytes(4 * nl, "little"), dtype=np.uint32) for a, _ in pairs])
    B = np.stack([np.frombuffer(b.to_bytes(4 * nl, "little"), dtype=np.uint32) for _, b in pairs])
    if len(pairs) == 1:
        return op, lambda: op.dmul_limbs(A[0], B[0], 2 * nl)
    return op, lambda: op.dmul_batch(A, B)


def cpu_baseline(N: int, pairs, budget_s: float):
    """The oracle on the host cores for about budget_s (bench's cpu_baseline key)."""
    threads = os.cpu_count() or 1
    op, run = _oracle_sample(N, pairs, threads)
    a, b = pairs[0]
    if op.dmul(a, b) != a * b:
        raise SystemExit("oracle mismatch")
    done, t0 = 0, time.perf_counter()
    while True:
        run()
        done += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s or done >= 1000:
            break
    prods = done * len(pairs)
    return {"value": round(2 * N * prods / dt / 1e9, 6), "unit": "Gbit/s", "cores": threads, "kind": "port",
            "sample": f"{prods} x 2^{N.bit_length() - 1}-bit products by oracle/dkss_oracle.c (C restatement of "
                      f"bigmul/dkss.py), {threads} OpenMP threads, {dt:.1f} s; the reference's own Python dmul "
                      f"takes 41 s per 2^20 multiply and 18 min per 2^24 multiply (BASELINE.md §2)"}


def run_reference(args):
    cfg = args.config
    N, pairs, seed, ones = CONFIGS[cfg]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    mode = mode_for(cfg, world, args.replicas)
    sample_pairs = min(pairs * (world if mode == "replicas" else 1), 16)
    sample = [operand_pair(N, seed, i, ones) for i in range(sample_pairs)]
    threads = os.cpu_count() or 1
    op, run = _oracle_sample(N, sample, threads)
    a, b = sample[0]
    if op.dmul(a, b) != a * b:
        raise SystemExit("oracle mismatch")
    for _ in range(args.warmup):
        run()
    budget = args.ref_budget
    times = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget:
            break
    dt = sum(times)
    value = 2 * N * sample_pairs * len(times) / dt / 1e9
    line = {"metric": METRIC, "value": round(value, 6), "unit": "Gbit/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "steps_timed": len(times), "warmup": args.warmup,
            "ms_per_step": round(1e3 * dt / len(times), 3), "higher_is_better": True, "scaling": scaling_for(mode),
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded random operands, SURVEY.md §8(d))",
            "config": config_dict(cfg, world, mode),
            "cpu_baseline": {"value": round(value, 6), "unit": "Gbit/s", "cores": threads, "kind": "port",
                             "sample": f"each step {sample_pairs} x 2^{N.bit_length() - 1}-bit products by "
                                       f"oracle/dkss_oracle.c (C restatement of bigmul/dkss.py) on {threads} host "
                                       f"threads; {len(times)} steps timed ({dt:.1f} s, budget {budget:.0f} s); "
                                       f"the reference's Python dmul takes 41 s per 2^20 multiply (BASELINE.md §2)"},
            "e2e": {"value": round(value, 6), "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# multi-rank plumbing

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """--gpus N without torchrun: start N ranks of this script under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


class Ranks:
    """rank / world / device of this process and the max-over-ranks reduction."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        # DKSS_BENCH_GLOO=1: gloo, every rank on the visible GPU(s) (orchestration check on 1 GPU)
        self.gloo = os.environ.get("DKSS_BENCH_GLOO", "0") not in ("", "0")
        if self.gloo:
            local %= max(1, torch.cuda.device_count())
        self.local = local
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        if self.world > 1:
            if self.gloo:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
        os.environ["DKSS_DEVICE"] = str(local)

    # every collective below is called by ALL ranks (never inside a rank-0-only branch)
    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device="cpu" if self.gloo else self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: int) -> int:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.int64, device="cpu" if self.gloo else self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return int(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def timed_steps(R: Ranks, step, steps: int, warmup: int, stream, per_step_barrier: bool = False):
    """W warm-up steps, then K steps each bracketed by CUDA events on `stream` with an L2 flush
    before it; returns (max-over-ranks device ms, clock summary, libdkss launches in the region)."""
    from paper_1503_04955_b200._native import kernel_launches

    torch = R.torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=R.dev)
    for _ in range(warmup):
        flush.zero_()
        if per_step_barrier:
            R.barrier()
        step()
    torch.cuda.synchronize(R.dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    clocks = ClockSampler(R.local)
    R.barrier()
    torch.cuda.synchronize(R.dev)
    n0 = kernel_launches()
    with clocks:
        for k in range(steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            if per_step_barrier:
                R.barrier()
            starts[k].record(stream)
            step()
            ends[k].record(stream)
        torch.cuda.synchronize(R.dev)
    launches = kernel_launches() - n0
    R.barrier()
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    return R.max(dev_ms), clocks.summary(), R.sum(launches)


def base_line(args, R: Ranks, mode: str, ms_per_step: float, value: float, clocks, launches) -> dict:
    return {"metric": METRIC, "value": round(value, 4), "unit": "Gbit/s", "impl": "ours", "n_gpus": R.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": scaling_for(mode), "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded random operands, SURVEY.md §8(d))",
            "config": config_dict(args.config, R.world, mode), "clocks": clocks,
            "gpu_launches": launches, "gpu_launches_per_step": round(launches / args.steps, 2)}


# ---------------------------------------------------------------------------
# our arm: split (one multiply over all ranks)

def run_split(args, R: Ranks):
    from paper_1503_04955_b200.dkss import set_device
    from paper_1503_04955_b200.fourstep import (DistExchange, PeerExchange, _operands, dmul_fourstep, make_rank,
                                                peer_capable, run_rank, run_rank_peer)
    from paper_1503_04955_b200.plan import dkss_select_params, ring_products_per_multiply

    torch = R.torch
    set_device(R.local)
    N, _, seed, ones = CONFIGS[args.config]
    a, b = operand_pair(N, seed, 0, ones)  # every rank holds the same operands
    plan = dkss_select_params(N)
    fs = make_rank(plan, R.rank, R.world, R.dev, ipc=args.exchange == "peer")
    A, B = _operands(plan, a, b, R.dev)
    exchange = args.exchange if (args.exchange == "alltoall" or peer_capable(fs)) else "alltoall"
    if exchange == "peer":
        px = PeerExchange(fs)

        def split_step():
            return run_rank_peer(fs, px, A, B)
    else:
        ex = DistExchange()

        def split_step():
            return run_rank(fs, ex, A, B)
    stream = torch.cuda.current_stream(R.dev)
    prod = split_step()
    torch.cuda.synchronize(R.dev)
    if R.rank == 0:
        c = int.from_bytes(prod.cpu().numpy().view("uint32").tobytes(), "little")
        if not gate_one(c, a, b, N):
            raise SystemExit("split product mismatch")
    R.barrier()
    max_ms, clocks, launches = timed_steps(R, split_step, args.steps, args.warmup, stream, per_step_barrier=True)
    ms_per_step = max_ms / args.steps
    e2e = []
    for _ in range(max(3, args.e2e_steps // 4)):
        R.barrier()
        t0 = time.perf_counter()
        dmul_fourstep(a, b, exchange=exchange)
        e2e.append(time.perf_counter() - t0)
    e2e_s = R.max(sorted(e2e)[len(e2e) // 2])
    if R.rank == 0:
        peak, peak_src = imad_peak()
        info = fs.stages.dp.info
        w_mul = ring_products_per_multiply(plan) * plan.m * plan.m * info["L"] * info["L"]
        per_gpu = w_mul / R.world / (ms_per_step * 1e-3)
        lay = fs.stages.layout(R.world)
        line = base_line(args, R, "split", ms_per_step, 2 * N / (ms_per_step * 1e-3) / 1e9, clocks, launches)
        line.update({
            "plan": plan_desc(plan),
            "exchange": exchange,
            "exchange_bytes_per_rank": 3 * 4 * lay["block_words"] * (R.world - 1) // R.world,
            "roofline": {"bound": "imad", "achieved": round(per_gpu / 1e12, 4), "peak": round(peak / 1e12, 4),
                         "unit": "T limb-products/s per GPU", "frac": round(per_gpu / peak, 4), "traffic": None,
                         "kernel": "whole split multiply (per GPU, exchanges included)", "peak_source": peak_src},
            "e2e": {"value": round(2 * N / e2e_s / 1e9, 4), "unit": "Gbit/s", "ms": round(e2e_s * 1e3, 3),
                    "h2d_bytes_per_step": 2 * A.numel() * 4 * R.world, "d2h_bytes_per_step": fs.prod.numel() * 4,
                    "api": "paper_1503_04955_b200.fourstep.dmul_fourstep(int, int) on every rank"},
        })
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm: one GPU, replicas, or the sharded batch

def plan_desc(plan) -> dict:
    return {"M": plan.M, "m": plan.m, "u": plan.u, "d": plan.d, "p_bits": plan.p.bit_length(), "levels": plan.levels,
            "base": plan.base_len}


def gate_one(c: int, a: int, b: int, N: int) -> bool:
    if N <= FULL_CHECK_MAX_BITS:
        return c == a * b
    return residues_ok(c, a, b, check_primes(64))


def run_local(args, R: Ranks, mode: str):
    import numpy as np

    from paper_1503_04955_b200.dkss import device_plan, dmul, dmul_many, set_device
    from paper_1503_04955_b200.parallel import shard_range
    from paper_1503_04955_b200.plan import dkss_select_params, ring_products_per_multiply
    from paper_1503_04955_b200.words import int_to_u32, u32_to_int

    torch = R.torch
    set_device(R.local)
    N, pairs_total, seed, ones = CONFIGS[args.config]
    if mode == "shard":
        lo, hi = shard_range(pairs_total, R.rank, R.world)
        idx = list(range(lo, hi))
    elif mode == "replicas":
        idx = [R.rank]  # rank r multiplies pair r of the seed's sequence
    else:
        idx = [0]
    pairs = [operand_pair(N, seed, i, ones) for i in idx]
    batch = len(pairs)
    plan = dkss_select_params(N)
    dp = device_plan(plan, R.local)
    info = dp.info
    nl, npl = info["operand_limbs"], info["product_limbs"]
    dA = torch.from_numpy(np.stack([int_to_u32(a, nl) for a, _ in pairs]).view(np.int32)).to(R.dev)
    dB = torch.from_numpy(np.stack([int_to_u32(b, nl) for _, b in pairs]).view(np.int32)).to(R.dev)
    dC = torch.zeros((batch, npl), dtype=torch.int32, device=R.dev)
    stream = torch.cuda.current_stream(R.dev)
    sp = stream.cuda_stream

    def step():
        dp.mul_device(batch, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), npl, sp)

    # correctness gate: every product of this rank (bigmul/bench.py:66-68)
    step()
    torch.cuda.synchronize(R.dev)
    C = dC.cpu().numpy().view(np.uint32)
    if batch == 1:
        ok = gate_one(u32_to_int(C[0]), *pairs[0], N)
        gate = "full a*b" if N <= FULL_CHECK_MAX_BITS else "residues mod 64 seeded 62-bit primes"
    else:
        primes = check_primes(8)
        full = set(range(0, batch, max(1, batch // 8))) | {batch - 1}
        ok = all(residues_ok(u32_to_int(C[i]), a, b, primes) for i, (a, b) in enumerate(pairs))
        ok = ok and all(u32_to_int(C[i]) == pairs[i][0] * pairs[i][1] for i in full)
        gate = (f"all {pairs_total} products by residues mod 8 seeded 62-bit primes, "
                f"{len(full) * R.world} in full against a*b")
    if not R.sum(0 if ok else 1) == 0:
        raise SystemExit("product mismatch in the correctness gate")

    max_ms, clocks, launches = timed_steps(R, step, args.steps, args.warmup, stream)
    ms_per_step = max_ms / args.steps
    products = (pairs_total if mode == "shard" else R.world) * args.steps
    value = 2 * N * products / (max_ms * 1e-3) / 1e9

    # per-launch profile (CUDA events between the same launches, un-graphed)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=R.dev)
    prof_runs = []
    for _ in range(5):
        flush.zero_()
        prof_runs.append(dp.profile_device(batch, dA.data_ptr(), dB.data_ptr(), nl, dC.data_ptr(), sp))
    del flush
    per_kind = {}
    for run in prof_runs[1:]:
        for kind, ms, work, nbytes in run:
            d = per_kind.setdefault(kind, {"ms": 0.0, "work": 0, "bytes": 0, "launches": 0})
            d["ms"] += ms
            d["work"] += work
            d["bytes"] += nbytes
            d["launches"] += 1
    nprof = len(prof_runs) - 1
    dom = max(per_kind, key=lambda k: per_kind[k]["ms"])
    dk = per_kind[dom]
    peaks = (imad_peak(), tc_i8_peak(), hbm_peak())
    roofs = {k: kernel_roofline(k, v["work"] // nprof, v["bytes"] // nprof, v["ms"] / nprof, peaks)
             for k, v in per_kind.items()}
    rp = ring_products_per_multiply(plan)
    w_mul = rp * plan.m * plan.m * info["L"] * info["L"]
    traffic, pipe_pct = None, None
    tpath = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            nt = json.load(f).get(args.config, {})
        traffic = nt.get(dom)
        pipe_pct = nt.get("fmaheavy_pct", {}).get(dom)

    # end to end through the public API (Python ints in, Natural out; H2D + D2H inside):
    # dmul for one product, dmul_many for this rank's pairs
    if batch == 1:
        def e2e_call():
            return [dmul(*pairs[0])]  # -> Natural, as the reference's dmul returns
    else:
        def e2e_call():
            return dmul_many(pairs)
    r = e2e_call()
    if any(r[i].to_int() != pairs[i][0] * pairs[i][1] for i in (0, len(r) - 1)):
        raise SystemExit("e2e product mismatch")
    del r
    e2e_times = []
    for _ in range(max(3, args.e2e_steps if batch == 1 else args.e2e_steps // 4)):
        R.barrier()
        t0 = time.perf_counter()
        e2e_call()
        e2e_times.append(time.perf_counter() - t0)
    e2e_times.sort()
    e2e_s = R.max(e2e_times[len(e2e_times) // 2])

    # the thesis's comparison baseline on the same operands: SMUL device time and T_DMUL / T_SMUL
    # (bigmul/bench.py:80-91), L2 flushed before every call
    smul_line = None
    if R.rank == 0:
        try:
            smul_line = smul_compare(torch, R, N, batch, dA, dB, nl, sp, stream, pairs[0], ms_per_step)
        except Exception as e:  # the headline does not depend on it; say why it is missing
            smul_line = {"unavailable": repr(e)[:200]}

    cpu = None
    if R.rank == 0 and R.world == 1 and not args.no_cpu:
        cpu = cpu_baseline(N, pairs[:1] if batch == 1 else pairs[:16], args.cpu_budget)

    if R.rank == 0:
        line = base_line(args, R, mode, ms_per_step, value, clocks, launches)
        # the step's roofline time: every kernel at its own bound (tensor / IMAD / HBM), summed
        t_roof = sum(r["t_roof_ms"] for r in roofs.values())
        prof_ms = sum(v["ms"] for v in per_kind.values()) / nprof
        dr = roofs[dom]
        line.update({
            "plan": plan_desc(plan), "gate": gate,
            "roofline": {"bound": dr["bound"], "achieved": dr["achieved"], "peak": dr["peak"], "unit": dr["unit"],
                         "frac": dr["frac"], "traffic": traffic, "kernel": dom,
                         "peak_source": {"imad": peaks[0][1], "tensor": peaks[1][1], "hbm": peaks[2][1]},
                         "ncu_fmaheavy_pct": pipe_pct,  # IMAD.WIDE pipe busy, from the committed ncu capture
                         "work_per_launch": dk["work"] // max(1, dk["launches"]),
                         "bytes_per_launch": dk["bytes"] // max(1, dk["launches"]),
                         "step_roofline_ms": round(t_roof, 5),
                         "step_frac": round(t_roof / prof_ms, 4) if prof_ms > 0 else None},
            "kernels": {k: {"ms_per_step": round(v["ms"] / nprof, 5), "launches_per_step": v["launches"] // nprof,
                            "work": v["work"] // nprof, "bytes": v["bytes"] // nprof, **roofs[k]}
                        for k, v in per_kind.items()},
            "ring_products_per_mul": rp, "w_mul_limb_products": w_mul,
            "e2e": {"value": round(2 * N * len(pairs) * R.world / e2e_s / 1e9, 4), "unit": "Gbit/s",
                    "ms": round(e2e_s * 1e3, 4), "e2e_over_device": round(e2e_s * 1e3 / ms_per_step, 3),
                    "h2d_bytes_per_step": 2 * nl * 4 * batch * R.world, "d2h_bytes_per_step": npl * 4 * batch * R.world,
                    "api": "paper_1503_04955_b200.dmul(int, int) -> Natural" if batch == 1 else
                           "paper_1503_04955_b200.dmul_many([(int, int)] * pairs) -> [Natural] on every rank"},
            "smul": smul_line,
        })
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)


def smul_compare(torch, R, N, batch, dA, dB, nl, sp, stream, pair0, ms_per_step):
    import numpy as np

    from paper_1503_04955_b200.smul import device_plan_for
    from paper_1503_04955_b200.words import u32_to_int

    splan, sdp = device_plan_for(2 * N, 64)
    snc = sdp.product_limbs
    dS = torch.zeros((batch, snc), dtype=torch.int32, device=R.dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=R.dev)

    def sstep():
        sdp.mul_device(batch, dA.data_ptr(), dB.data_ptr(), nl, dS.data_ptr(), snc, sp)

    sstep()
    torch.cuda.synchronize(R.dev)
    S0 = dS[0].cpu().numpy().view(np.uint32)
    sts = []
    for i in range(8):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sstep()
        e1.record(stream)
        torch.cuda.synchronize(R.dev)
        if i >= 2:
            sts.append(e0.elapsed_time(e1))
    s_ms = float(np.median(sts))
    return {"ms_per_step": round(s_ms, 5), "gbit_s": round(2 * N * batch / (s_ms * 1e-3) / 1e9, 4),
            "dmul_over_smul": round(ms_per_step / s_ms, 3), "exact": gate_one(u32_to_int(S0), *pair0, N),
            "plan": {"m": splan.m, "K": splan.K, "s": splan.s}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--replicas", action="store_true",
                    help="single-multiply configs at N > 1: independent replicas instead of the four-step split")
    ap.add_argument("--exchange", default="peer", choices=["peer", "alltoall"],
                    help="four-step split: exchange fused into the phase kernels' stores over CUDA IPC peer "
                         "memory (default), or NCCL all-to-all + re-layout kernels")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--ref-budget", type=float, default=150.0, help="seconds of timed oracle work, reference arm")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    R = Ranks()
    try:
        if R.world != args.gpus and R.rank == 0:
            print(f"note: --gpus {args.gpus} but WORLD_SIZE={R.world}; measuring {R.world} ranks", file=sys.stderr)
        mode = mode_for(args.config, R.world, args.replicas)
        if mode == "split":
            run_split(args, R)
        else:
            run_local(args, R, mode)
    finally:
        R.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
