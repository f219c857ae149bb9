"""DKSS multiplication on B200 behind the reference's Python API.

Public entry points keep the reference signatures (BASELINE.json north_star:
"The Python package's public multiply entry points keep their signatures, so
the build is a drop-in"):

* ``dmul(a, b, thresholds=None, arena=None) -> Natural``   -- bigmul/dkss.py:520-548
* ``dkss_encode(a, plan, arena=None)``                      -- bigmul/dkss.py:381-398
* ``dkss_fft(v, plan, table=None, arena=None, base_pow=1)`` -- bigmul/dkss.py:443-495
* ``r_mul(x, y, plan, table=None, arena=None)``             -- bigmul/dkss.py:401-420
* ``dkss_decode(v, plan, arena=None) -> Natural``           -- bigmul/dkss.py:498-513

Host work is parameter selection (plan.py, identical to the reference) and
int <-> u32-limb conversion; every arithmetic step runs in libdkss.so on the
GPU (no CPU fallback -- a missing library raises).  The stage functions accept
and return the reference's list-of-lists representation; the ``*_limbs``
variants take numpy uint32[2M][m][L] arrays and skip the Python int boxing.
"""

from __future__ import annotations

import os
import threading

import numpy as np

from ._native import DKSS_DIGITS_TRUSTED, DevicePlan, pinned_empty
from .plan import DkssPlan, dkss_select_params, ring_products_per_multiply, twiddle_count
from .words import (Natural, ScratchArena, as_natural, current_arena, foreign_natural, int_to_u32, pylong_digits,
                    u32_to_int, word_bits, words_to_int, PYLONG_DIGIT_BITS)

# The reference hands products below 2048 result bits to smul (bigmul/dkss.py:517,
# 533-535); here dmul always measures DKSS, so such inputs run through DKSS on the GPU
# with the plan for N = _MIN_PLAN_BITS (any input below 2^N fits a plan for N).
_MIN_DKSS_BITS = 2048
_MIN_PLAN_BITS = 1024

_dev_lock = threading.Lock()
_dev_plans: dict = {}
_host_plans: dict = {}


def _plan_for(N: int, w: int) -> DkssPlan:
    """Host plan for inputs below 2^N at word size w, built (and verified) once.

    The reference re-runs dkss_select_params on every dmul (the rho-power table is
    cached in make_plan, bigmul/dkss.py:220-233, but rho is re-verified each call);
    the plan is a pure function of (N, w), so caching it changes no result.
    """
    key = (N, w)
    with _dev_lock:
        pl = _host_plans.get(key)
    if pl is None:
        pl = dkss_select_params(N, w)
        with _dev_lock:
            if key not in _host_plans:
                _cache_put(_host_plans, key, pl)
    return pl


_device_ordinal: int | None = None


def _device() -> int:
    """GPU ordinal: set_device(), else DKSS_DEVICE read at the first call (default 0)."""
    global _device_ordinal
    if _device_ordinal is None:
        _device_ordinal = int(os.environ.get("DKSS_DEVICE", "0"))
    return _device_ordinal


def set_device(ordinal: int) -> None:
    """Select the GPU later multiplies of this process run on."""
    global _device_ordinal
    _device_ordinal = int(ordinal)


_MAX_PLANS = 32  # cached plans per kind; older entries are dropped (and freed when unreferenced)


def _cache_put(cache: dict, key, value):
    cache[key] = value
    while len(cache) > _MAX_PLANS:
        cache.pop(next(iter(cache)))


def plan_capacity(plan: DkssPlan) -> int:
    """Largest operand bit length the plan's geometry encodes: M coefficients of m/2 u-bit
    pieces (bigmul/dkss.py:381-398).  Every N the planner maps to (M, m, u) is at most this."""
    return plan.M * (plan.m // 2) * plan.u


def device_plan(plan: DkssPlan, device: int | None = None, lane: int = 0) -> DevicePlan:
    """Upload (once) and return the device plan for a host plan.

    Device plans are shared by every N with the same geometry (M, m, u, p): they are built for
    the geometry's capacity, so multiplying operands of many different sizes does not create
    a device plan (twiddle table + workspace) per size.  ``lane`` > 0 gives further handles of
    the same geometry (own stream and workspace) for concurrent host threads."""
    device = _device() if device is None else device
    key = (plan.M, plan.m, plan.u, plan.p, device) + ((lane,) if lane else ())
    with _dev_lock:
        dp = _dev_plans.get(key)
        if dp is None:
            dp = DevicePlan(plan_capacity(plan), plan.M, plan.m, plan.u, plan.p, plan.rho_powers, device)
            _cache_put(_dev_plans, key, dp)
        return dp


def clear_device_plans() -> None:
    with _dev_lock:
        _hot.clear()
        for dp in _dev_plans.values():
            dp.close()
        _dev_plans.clear()


def _L(plan: DkssPlan) -> int:
    return -(-plan.pz.bit_length() // 32)


def poly_to_limbs(poly, plan: DkssPlan) -> np.ndarray:
    """list[2M][m] of ints -> uint32[2M, m, L]"""
    L = _L(plan)
    raw = b"".join(int(c).to_bytes(4 * L, "little") for row in poly for c in row)
    return np.frombuffer(raw, dtype=np.uint32).reshape(len(poly), plan.m, L).copy()


def limbs_to_poly(arr: np.ndarray) -> list:
    n, m, L = arr.shape
    flat = arr.reshape(-1, L)
    vals = [int.from_bytes(row.tobytes(), "little") for row in flat]
    return [vals[i * m:(i + 1) * m] for i in range(n)]


# ---------------------------------------------------------------------------
# stages

def dkss_encode_limbs(a, plan: DkssPlan) -> np.ndarray:
    ai = as_natural(a).to_int()
    if plan.N and ai >= 1 << plan.N:
        raise ValueError("operand does not fit the plan")
    dp = device_plan(plan)
    return dp.encode(int_to_u32(ai, max(1, dp.info["operand_limbs"])))


def dkss_encode(a, plan: DkssPlan, arena: ScratchArena | None = None):
    arena = arena or current_arena()
    arena.alloc_words(2 * plan.M * plan.oclen)
    return limbs_to_poly(dkss_encode_limbs(a, plan))


def dkss_fft_limbs(polys: np.ndarray, plan: DkssPlan) -> np.ndarray:
    return device_plan(plan).fft(polys)


def dkss_fft(v, plan: DkssPlan, table=None, arena: ScratchArena | None = None, base_pow: int = 1) -> None:
    """In place: v[i] <- a(rho^i) (natural order), like the reference."""
    length = len(v)
    if length & (length - 1):
        raise ValueError("transform length must be a power of 2")
    if base_pow != 1 or length != 2 * plan.M:
        raise ValueError("the device transform evaluates the full length-2M transform (base_pow=1)")
    out = dkss_fft_limbs(poly_to_limbs(v, plan), plan)
    plan.ks_calls += twiddle_count(plan)
    v[:] = limbs_to_poly(out)


def r_mul_limbs(x: np.ndarray, y: np.ndarray, plan: DkssPlan) -> np.ndarray:
    return device_plan(plan).rmul(x, y)


def r_mul(x, y, plan: DkssPlan, table=None, arena: ScratchArena | None = None):
    plan.ks_calls += 1
    L = _L(plan)
    xa = poly_to_limbs([x], plan)
    ya = poly_to_limbs([y], plan)
    del L
    return limbs_to_poly(r_mul_limbs(xa, ya, plan))[0]


def dkss_decode_limbs(v: np.ndarray, plan: DkssPlan, nout: int) -> np.ndarray:
    return device_plan(plan).decode(v, nout)


def dkss_decode(v, plan: DkssPlan, arena: ScratchArena | None = None) -> Natural:
    dp = device_plan(plan)
    limbs = dkss_decode_limbs(poly_to_limbs(v, plan), plan, dp.info["product_limbs"])
    value = u32_to_int(limbs)
    return Natural.from_int(value) if value else Natural([0])


# ---------------------------------------------------------------------------
# the multiply

def _caller(*xs):
    """(Natural class to return, word size) of a call: the reference's own class and word size
    when it handed in its bigmul.words.Natural (the reference's mul, run_bench and lucas_lehmer
    convert operands before calling ALGORITHMS[...], bigmul/dispatch.py:30-36,
    bigmul/bench.py:35-64, 210-213), else (None, this package's word size)."""
    for x in xs:
        fw = foreign_natural(x)
        if fw is not None:
            return fw
    return None, word_bits()


def _deliver(n: Natural, cls):
    """The product as the caller's Natural class (same words, same word size)."""
    return n if cls is None else cls(n.words)


def _as_int_len(x, w: int):
    """(value, word length at word size w) exactly as as_natural(x) would give
    (bigmul/words.py:112-117); a foreign Natural's words are read at its own word size w."""
    if type(x) is int:  # the common case first
        if x < 0:
            raise ValueError("Natural is nonnegative")
        return x, max(1, -(-x.bit_length() // w))
    if isinstance(x, Natural):
        return x.to_int(w), len(x)
    if foreign_natural(x) is not None:
        ws = x.words
        return words_to_int(ws, w), len(ws)
    if isinstance(x, int) and not isinstance(x, bool):
        if x < 0:
            raise ValueError("Natural is nonnegative")
        return x, max(1, -(-x.bit_length() // w))
    n = as_natural(x)
    return n.to_int(), len(n)


def _digits(x, value: int):
    """(keepalive, host address, digit count, digit bits) of an operand for dkss_mul_digits."""
    if isinstance(x, Natural) and x._words is None and x._w == word_bits():
        arr = np.ascontiguousarray(x._limbs, dtype=np.uint32)
        return arr, arr.ctypes.data, arr.size, 32
    d = pylong_digits(value)
    if d is not None:  # CPython keeps every digit below 2^30: no scan needed
        return value, d[0], d[1], PYLONG_DIGIT_BITS | DKSS_DIGITS_TRUSTED
    arr = int_to_u32(value, max(1, -(-value.bit_length() // 32)))
    return arr, arr.ctypes.data, arr.size, 32


_hot: dict = {}


def _hot_plan(N: int, w: int):
    """(plan, device plan, operand limbs, product limbs, workspace words, r_mul count), cached
    per (N, w, device) so a multiply does no per-call plan bookkeeping."""
    key = (N, w, _device())
    ent = _hot.get(key)
    if ent is None:
        plan = _plan_for(N, w)
        dp = device_plan(plan, key[2])
        info = dp.info
        ent = (plan, dp, info["operand_limbs"], info["product_limbs"], info["footprint_bytes"],
               ring_products_per_multiply(plan))
        with _dev_lock:
            _cache_put(_hot, key, ent)
    return ent


def dmul(a, b, thresholds=None, arena: ScratchArena | None = None) -> Natural:
    """Full product via DKSS on the GPU (bigmul/dkss.py:520-548).

    a, b: int, this package's Natural or the reference's bigmul.words.Natural; the result is a
    Natural of len(a) + len(b) words of the caller's class and word size.  ``arena`` records the
    device bytes the multiply holds (dkss_plan_info.footprint_bytes)."""
    cls, w = _caller(a, b)
    ai, la = _as_int_len(a, w)
    bi, lb = _as_int_len(b, w)
    arena = arena or current_arena()
    outlen = max(1, la + lb)
    if ai == 0 or bi == 0:
        return _deliver(Natural([0] * outlen), cls)
    n_bits = max(ai.bit_length(), bi.bit_length())
    plan, dp, nl, npl, footprint, rp = _hot_plan(max(n_bits, _MIN_PLAN_BITS), w)
    nc = max(npl, -(-outlen * w // 32))
    mark = arena.acquire()
    try:
        arena.alloc_words(-(-footprint * 8 // w))
        ka, pa, na, ba = _digits(a, ai)
        kb, pb, nb, bb = (ka, pa, na, ba) if b is a else _digits(b, bi)
        if ba == bb:
            c = dp.mul_digits(pa, na, pb, nb, ba, nc)
        else:
            c = dp.mul_limbs(int_to_u32(ai, nl), int_to_u32(bi, nl), nc)
        del ka, kb
    finally:
        arena.release(mark)
    plan.ks_calls += rp
    return _deliver(Natural._from_u32(c, outlen, w), cls)


_PIPE_MIN_PAIRS = 64   # batches at least this large run as chunks on two device lanes
# chunks (at least 64 pairs each) dealt round-robin to device lanes; measured at 1024 x 2^18
# (tools/batch_lanes_probe.py, e2e ms): 2 lanes x 2 chunks 9.8, 2 x 4 9.4, 3 x 6 8.4, 4 x 4 8.7,
# 4 x 8 8.1, 4 x 16 8.2, 8 x 16 8.3
_PIPE_CHUNKS = 8
_PIPE_LANES = 4
_pipe_pool = None


def _pipelined_batch(plan, da, db, digit_bits: int, nc: int) -> np.ndarray:
    """The batch as up to _PIPE_CHUNKS chunks on up to _PIPE_LANES device plans (own stream and
    workspace each), one host thread per lane: a chunk's host staging, H2D and D2H overlap the
    other lanes' device work (the C call releases the GIL).  Same products as one batch call."""
    global _pipe_pool
    from concurrent.futures import ThreadPoolExecutor

    n = len(da)
    nchunks = max(2, min(_PIPE_CHUNKS, n // _PIPE_MIN_PAIRS))
    lanes = max(1, min(_PIPE_LANES, nchunks))
    if _pipe_pool is None or _pipe_pool._max_workers < lanes:
        _pipe_pool = ThreadPoolExecutor(max_workers=lanes, thread_name_prefix="dkss-lane")
    step = -(-n // nchunks)
    chunks = [(i, min(n, i + step)) for i in range(0, n, step)]
    out = pinned_empty((n, nc))  # the lanes' products land here straight from the device
    device = _device()

    def lane_work(lane):
        dpl = device_plan(plan, device, lane)
        for k in range(lane, len(chunks), lanes):
            lo, hi = chunks[k]
            dpl.mul_batch_digits([d[1] for d in da[lo:hi]], [d[2] for d in da[lo:hi]], [d[1] for d in db[lo:hi]],
                                 [d[2] for d in db[lo:hi]], digit_bits, nc, out=out[lo:hi])

    futs = [_pipe_pool.submit(lane_work, lane) for lane in range(lanes)]
    for f in futs:
        f.result()
    return out


def dmul_many(pairs, thresholds=None) -> list:
    """Independent products sharing one plan, batched in one device call (config 3).

    Returns one Natural per pair, as dmul would (len(a) + len(b) words)."""
    pairs = list(pairs)
    if not pairs:
        return []
    cls, w = _caller(*pairs[0])
    vals = [(_as_int_len(a, w), _as_int_len(b, w)) for a, b in pairs]
    n_bits = max(max(ai.bit_length(), bi.bit_length()) for (ai, _), (bi, _) in vals)
    plan = _plan_for(max(n_bits, _MIN_PLAN_BITS), w)
    dp = device_plan(plan)
    nl = dp.info["operand_limbs"]
    lens = [max(1, la + lb) for (_, la), (_, lb) in vals]
    nc = max(dp.info["product_limbs"], -(-max(lens) * w // 32))
    da = [_digits(a, ai) for (a, _), ((ai, _), _) in zip(pairs, vals)]
    db = [_digits(b, bi) for (_, b), (_, (bi, _)) in zip(pairs, vals)]
    bits = {d[3] for d in da} | {d[3] for d in db}
    if len(bits) == 1 and len(pairs) >= _PIPE_MIN_PAIRS:
        C = _pipelined_batch(plan, da, db, bits.pop(), nc)
    elif len(bits) == 1:
        C = dp.mul_batch_digits([d[1] for d in da], [d[2] for d in da], [d[1] for d in db], [d[2] for d in db],
                                bits.pop(), nc)
    else:
        A = np.stack([int_to_u32(ai, nl) for (ai, _), _ in vals])
        B = np.stack([int_to_u32(bi, nl) for _, (bi, _) in vals])
        C = dp.mul_batch(A, B, nc)
    del da, db
    plan.ks_calls += len(pairs) * ring_products_per_multiply(plan)
    return [_deliver(Natural._from_u32(C[i], lens[i], w), cls) for i in range(len(pairs))]
