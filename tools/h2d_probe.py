"""PCIe probe for the host digits path: H2D of an operand-sized pinned buffer alone, with a
concurrent multi-threaded host memcpy (the staging of the next operand), from a write-combined
pinned buffer, and the host memcpy rate itself.

  python tools/h2d_probe.py [--mb 2.24] [--reps 20]
"""
import argparse
import threading
import time

import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--mb", type=float, default=2.24)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
n = int(args.mb * (1 << 20)) // 4
dev = torch.empty(n, dtype=torch.int32, device="cuda")
pin = torch.empty(n, dtype=torch.int32).pin_memory()
src = np.random.randint(0, 1 << 30, size=n, dtype=np.int32)
dst2 = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
s = torch.cuda.Stream()


def h2d(buf):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        dev.copy_(buf, non_blocking=True)
        e1.record(s)
    return e0, e1


def med(xs):
    xs = sorted(xs)
    return round(xs[len(xs) // 2], 1)


out = {}
t = []
for _ in range(args.reps):
    e0, e1 = h2d(pin)
    torch.cuda.synchronize()
    t.append(e0.elapsed_time(e1) * 1e3)
out["h2d_alone_us"] = med(t)


def hostcopy(k=8):
    ch = -(-n // k)
    ths = [threading.Thread(target=lambda i=i: np.copyto(dst2[i * ch:(i + 1) * ch], src[i * ch:(i + 1) * ch])) for i in range(k)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()


t, th_t = [], []
for _ in range(args.reps):
    e0, e1 = h2d(pin)
    t0 = time.perf_counter()
    hostcopy()
    th_t.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    t.append(e0.elapsed_time(e1) * 1e3)
out["h2d_with_host_copy_us"] = med(t)
out["host_copy_8thr_us"] = med(th_t)
th_t = []
for _ in range(args.reps):
    t0 = time.perf_counter()
    np.copyto(dst2, src)
    th_t.append((time.perf_counter() - t0) * 1e6)
out["host_copy_1thr_us"] = med(th_t)
out["bytes"] = 4 * n
import os
out["cpus"] = os.cpu_count()
print(out)
