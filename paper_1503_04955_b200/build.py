"""Build libdkss.so (sm_100a) in-tree: paper_1503_04955_b200/_lib/libdkss.so.

nvcc -gencode arch=compute_100a,code=sm_100a, one translation unit per (m, L)
kernel instantiation plus the host/C-ABI unit, compiled in parallel and linked
into one shared library.  Incremental: an object is rebuilt only when a source
or header is newer.  ``python -m paper_1503_04955_b200.build [-j N] [--force]``.
"""

from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# DKSS_VARIANT=name builds an experiment library _lib/libdkss_<name>.so with the extra
# nvcc flags in DKSS_EXTRA_FLAGS (loaded when DKSS_LIB points at it); default: the product
VARIANT = os.environ.get("DKSS_VARIANT", "")
OBJ = os.path.join(HERE, "_build" + (f"_{VARIANT}" if VARIANT else ""))
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, f"libdkss_{VARIANT}.so" if VARIANT else "libdkss.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# experiment libraries also read the DKSS_* environment switches (csrc/dkss_capi.cu DKSS_KNOB);
# the product library reads none
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE,
         *(["-DDKSS_EXPERIMENTS"] if VARIANT else []), *os.environ.get("DKSS_EXTRA_FLAGS", "").split()]

INSTANCES = [(m, L) for m in (8, 16, 32) for L in (2, 3, 4, 5, 6)]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _units():
    hdrs = _headers()
    units = [(os.path.join(OBJ, "dkss_capi.o"), os.path.join(CSRC, "dkss_capi.cu"), [], hdrs)]
    for m, L in INSTANCES:
        units.append((os.path.join(OBJ, f"dkss_inst_m{m}_L{L}.o"), os.path.join(CSRC, "dkss_inst.cu"),
                      [f"-DINST_MM={m}", f"-DINST_L={L}"], hdrs))
    return units


def build(jobs: int | None = None, force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    todo = [u for u in _units() if force or _stale(u[0], [u[1]] + u[3])]

    def compile_one(u):
        obj, src, defs, _ = u
        cmd = [NVCC, *ARCH, *FLAGS, *defs, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {os.path.basename(obj)}:\n{r.stderr[-4000:]}")
        return obj

    if todo:
        with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
            list(ex.map(compile_one, todo))
    objs = [u[0] for u in _units()]
    if force or todo or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args(argv)
    print(build(a.j, a.force, a.v))


if __name__ == "__main__":
    sys.exit(main())
