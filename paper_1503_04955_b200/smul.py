"""Schoenhage-Strassen multiplication (SMUL) on the GPU -- the reference's comparison
baseline for DKSS (bigmul/smul.py).

Host side: the plan selection of bigmul/smul.py:20-153 restated (candidate (m, K) per FFT
depth, the cost model, near-ties to the shorter FFT), so ``smul_select_params`` returns the
reference's plan field for field.  Device side (include/smul.h): the outermost cyclic level
(bigmul/smul.py:219-271, 286-300) -- encode, forward FFTs over Z/(2^K+1), pointwise
products, inverse FFT with the 2^-m normalisation, overlap-add -- as sm_100a kernels.

Deliberate differences, none visible in results (every plan computes a*b exactly): the
pointwise products are computed directly on the GPU (the reference recurses into smul or
Toom-3, bigmul/smul.py:206-216; both give the same residue); products below 512 bits also
go through a plan (the reference hands them to t3mul, bigmul/smul.py:294-295); and the
device picks its plan from the reference's candidate list with its own cost model
(``device_select_params``).  ``smul_select_params`` is the reference's choice, field for
field, and the stage functions run on any outermost plan with K a multiple of 32.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from math import gcd

import numpy as np

from ._native import SmulDevicePlan
from .dispatch import ThresholdTable, default_thresholds
from .words import Natural, ScratchArena, current_arena, int_to_u32, word_bits

DEVICE_K_MAX = 32768  # include/smul.h: K up to 32768 bits


@dataclass(frozen=True)
class SmulPlan:
    """bigmul/smul.py:20-30."""

    N: int          # products come out mod 2^N + 1
    m: int          # FFT depth
    n: int          # FFT length 2^m
    s: int          # input bits per coefficient, N == s * n
    K: int          # coefficient ring bits
    omega_exp: int  # omega = 2^omega_exp
    theta_exp: int  # 0 on the cyclic outermost level
    outermost: bool
    w: int

    def fe_word_count(self) -> int:
        return self.K // self.w + 1  # bigmul/fermat.py:52-55

    def validate(self) -> "SmulPlan":
        """The checks of bigmul/smul.py:35-52."""
        if self.s * self.n != self.N:
            raise ValueError("N must equal s * 2^m")
        if self.K < self.m + 2 * self.s + 1:
            raise ValueError("K below the convolution bound m + 2s + 1")
        if self.K % self.w:
            raise ValueError("K not word aligned")
        if self.outermost:
            if (2 * self.K) % self.n:
                raise ValueError("outermost level needs n | 2K")
        else:
            if self.K % self.n:
                raise ValueError("negacyclic level needs n | K")
            if self.theta_exp * 2 != self.omega_exp:
                raise ValueError("theta^2 must equal omega")
        if pow(2, self.omega_exp * self.n // 2, (1 << self.K) + 1) != (1 << self.K):
            raise ValueError("omega is not a principal n-th root")
        return self


def _round_up(v: int, a: int) -> int:
    return (v + a - 1) // a * a


def smul_plan_candidates(N: int, outermost: bool, w: int | None = None, validate: bool = True) -> list:
    """Every feasible (m, K) for an N-bit modulus (bigmul/smul.py:75-105): per depth m the
    smallest admissible K, then the next power of two if it is at most twice that.
    ``validate=False`` skips the per-plan checks (a modular power over 2^K + 1 each; the
    candidates satisfy them by construction) -- the device planner's fast path."""
    w = word_bits() if w is None else w
    out = []
    for m in range(1, 27):
        n = 1 << m
        if not outermost and N % n:
            continue
        s = (N + n - 1) // n
        k_floor = m + 2 * s + 1
        step = max(n // 2 if outermost else n, 1)
        align = step * w // gcd(step, w)
        k_min = _round_up(k_floor, align)
        if k_min > 64 * N + 64:
            continue
        ks = [k_min]
        k_pow = 1 << (k_min - 1).bit_length()
        if k_pow != k_min and k_pow % align == 0 and k_pow <= 2 * k_min:
            ks.append(k_pow)
        for K in ks:
            if not outermost and K >= N:
                continue
            if outermost:
                om, th = 2 * K // n, 0
            else:
                om, th = 2 * (K // n), K // n
            p = SmulPlan(s * n, m, n, s, K, om, th, outermost, w)
            out.append(p.validate() if validate else p)
        if n >= 2 * k_floor and n >= 2 * w:
            break
    return out


def _plan_cost(p: SmulPlan) -> float:
    """bigmul/smul.py:121-125: three transforms, n pointwise products, linear work."""
    return 4.5 * p.n * p.m * p.K + p.n * (p.K ** 1.465) + 10 * p.n * p.K


def smul_select_params(N: int, outermost: bool, w: int | None = None,
                       table: ThresholdTable | None = None) -> SmulPlan:
    """bigmul/smul.py:128-153: a depth pinned by the table's smul_fft_m bucket, else the
    cheapest plan by the cost model with ties within 5% going to the shorter FFT."""
    w = word_bits() if w is None else w
    table = table or default_thresholds()
    cands = smul_plan_candidates(N, outermost, w)
    if not cands:
        raise ValueError(f"no feasible Schoenhage-Strassen plan for N={N}")
    if outermost:
        forced = table.smul_fft_m.get(max(0, (N // w).bit_length() - 1))
        if forced is not None:
            for p in cands:
                if p.m == forced:
                    return p
    best = min(cands, key=_plan_cost)
    limit = 1.05 * _plan_cost(best)
    for p in sorted(cands, key=lambda q: q.n):
        if _plan_cost(p) <= limit:
            return p
    return best


_lock = threading.Lock()
_dev: dict = {}
_MAX = 32


def _device_cost(p: SmulPlan) -> float:
    """Device cost of a candidate: transform limb work (a lane holds 1, 2, 3, 4, 6, 8, 16 or
    32 limbs, ~8 instructions per limb per butterfly), the schoolbook pointwise products, and
    a penalty when the n products cannot fill the 148 SMs."""
    kw = p.K // 32
    q = next(x for x in (1, 2, 3, 4, 6, 8, 16, 32, 64) if 32 * x >= kw)  # limbs per lane, csrc/smul_capi.cuh
    work = 1.5 * p.n * p.m * 32 * q * 8 + p.n * kw * kw
    full = 1.0 if kw == 32 * q else 1.2  # kernels with every lane slot live skip the bounds checks
    return full * work / min(1.0, p.n / 2048)


def device_select_params(n0: int, w: int, table: ThresholdTable | None = None) -> SmulPlan:
    """The plan the device runs a product of n0 bits on.  The result does not depend on the
    plan (every plan computes a*b), so the device picks its own from the reference's
    candidate list (bigmul/smul.py:75-105) by `_device_cost` -- the reference's cost model
    (bigmul/smul.py:121-125) prices a recursive Toom-3 pointwise product and favours few,
    wide coefficients (2^20 x 2^20 bits: n = 512, K = 8448), where a GPU wants many narrow
    ones (n = 2048-4096, K = 2048-3072).  A depth pinned by the table is honoured."""
    table = table or default_thresholds()
    wd = max(w, 32)
    forced = table.smul_fft_m.get(max(0, (n0 // w).bit_length() - 1))
    if forced is not None:
        p = smul_select_params(n0, True, wd, table)
        if p.m == forced and p.K % 32 == 0 and p.K <= DEVICE_K_MAX:
            return p
    cands = [p for p in smul_plan_candidates(n0, True, wd, validate=False) if p.K % 32 == 0 and p.K <= DEVICE_K_MAX]
    if not cands:
        raise ValueError(f"no device Schoenhage-Strassen plan for N={n0}")
    return min(cands, key=_device_cost)


_sel_cache: dict = {}


def device_plan_for(n0: int, w: int, table: ThresholdTable | None = None, device: int | None = None):
    """(host plan, device plan) for a product of n0 bits at word size w.  The selection is
    cached per (n0, w, pinned depth): enumerating the candidates validates every one with a
    modular power over 2^K + 1 (milliseconds at 2^20), far more than the multiply."""
    from .dkss import _device

    device = _device() if device is None else device
    table = table or default_thresholds()
    # nearby sizes share a plan: n0 rounded up to 1/32 of its octave (any plan with N >= n0
    # computes the product exactly)
    step = 1 << max(0, n0.bit_length() - 6)
    n0r = -(-n0 // step) * step
    key = (n0r, w, table.smul_fft_m.get(max(0, (n0 // w).bit_length() - 1)))
    plan = _sel_cache.get(key)
    if plan is None:
        plan = device_select_params(n0r, w, table)
        with _lock:
            _sel_cache[key] = plan
            while len(_sel_cache) > 1024:
                _sel_cache.pop(next(iter(_sel_cache)))
    return plan, _device_plan(plan, device)


def _device_plan(plan: SmulPlan, device: int):
    if not plan.outermost:
        raise ValueError("the device runs the outermost (cyclic) level only")
    key = (plan.N, plan.m, plan.s, plan.K, plan.omega_exp, device)
    with _lock:
        dp = _dev.get(key)
        if dp is None:
            dp = SmulDevicePlan(plan.N, plan.m, plan.s, plan.K, plan.omega_exp, device)
            _dev[key] = dp
            while len(_dev) > _MAX:
                # dropped, not closed: a thread may still be multiplying on the evicted plan;
                # SmulDevicePlan.__del__ frees it once the last reference goes
                _dev.pop(next(iter(_dev)))
    return dp


def smul(a, b, thresholds: ThresholdTable | None = None, arena: ScratchArena | None = None) -> Natural:
    """Full product via the outermost Schoenhage-Strassen level on the GPU
    (bigmul/smul.py:286-300): a Natural of len(a) + len(b) words."""
    from .dkss import _as_int_len, _caller, _deliver, _digits  # (value, word length) without a Natural

    arena = arena or current_arena()
    cls, w = _caller(a, b)  # the reference's Natural class and word size when it passed its own
    ai, la_w = _as_int_len(a, w)
    bi, lb_w = _as_int_len(b, w)
    outlen = max(1, la_w + lb_w)
    if ai == 0 or bi == 0:
        return _deliver(Natural([0] * outlen), cls)
    n0 = ai.bit_length() + bi.bit_length()
    plan, dp = device_plan_for(n0, w, thresholds)
    nc = max(1, -(-outlen * w // 32))
    la, lb = -(-ai.bit_length() // 32), -(-bi.bit_length() // 32)
    with arena.frame():
        arena.alloc_words(2 * plan.n * plan.fe_word_count() + plan.fe_word_count())  # bigmul/smul.py:232
        ka, pa, na, ba = _digits(a, ai)
        kb, pb, nb, bb = (ka, pa, na, ba) if b is a else _digits(b, bi)
        if ba == bb:  # CPython's own digits (or limbs) go straight to the device
            c = dp.mul_digits(pa, na, pb, nb, ba, nc)
        else:
            A = int_to_u32(ai, la)
            c = dp.mul_limbs(A, A if bi == ai else int_to_u32(bi, lb), nc)
        del ka, kb
    return _deliver(Natural._from_u32(c, outlen, w), cls)


def fft_eval_fermat(v: list, plan: SmulPlan, inverse: bool = False) -> None:
    """fft_eval(v, FermatRing(K, omega_exp, n)) in place on the GPU (bigmul/fft.py:70-109,
    bigmul/fermat.py:67-93): v holds n canonical residues in [0, 2^K], shuffled order in,
    natural order out; ``inverse`` uses omega^-1 (FermatRing.inverse_ring)."""
    from .dkss import _device

    dp = _device_plan(plan, _device())
    kw = plan.K // 32
    x = np.zeros((plan.n, kw), dtype=np.uint32)
    top = np.zeros(plan.n, dtype=np.uint32)
    mask = (1 << plan.K) - 1
    for i, val in enumerate(v):
        if not 0 <= val <= (1 << plan.K):
            raise ValueError("element not canonical in [0, 2^K]")
        top[i] = val >> plan.K
        x[i] = np.frombuffer((val & mask).to_bytes(4 * kw, "little"), dtype=np.uint32)
    dp.fft(x, top, inverse)
    for i in range(plan.n):
        v[i] = int.from_bytes(x[i].tobytes(), "little") | (int(top[i]) << plan.K)
