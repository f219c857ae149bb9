"""Lucas-Lehmer system test on the GPU DKSS multiply.

Restates the reference driver (bigmul/bench.py:187-217): ``lucas_lehmer(p, multiplier,
thresholds) -> (is_prime, residue64)`` with s_0 = 4, s <- (s^2 - 2) mod (2^p - 1) for p - 2
steps; residue64 = the low 64 bits of the final s, so one wrong bit anywhere in a multiply
scrambles it.  With ``multiplier="dmul"`` the whole loop runs on the device
(``dkss_lucas_lehmer``): every square goes through the DKSS pipeline in squaring mode (one
forward transform, pointwise squares, inverse, decode) and the reduction
mod 2^p - 1 and the "- 2" run in one more kernel; the state never leaves the GPU between
steps.  ``multiplier="smul"`` squares with the GPU Schoenhage-Strassen multiply and reduces
on the host; the reference's other rungs are out of scope here (dispatch.ALGORITHMS raises
NotImplementedError for them).
"""

from __future__ import annotations

from .dispatch import ALGORITHMS
from .dkss import _MIN_PLAN_BITS, _plan_for, device_plan
from .words import int_to_u32, u32_to_int, word_bits


def mersenne_reduce(x: int, p: int) -> int:
    """x mod 2^p - 1 by folding (bigmul/bench.py:187-194), canonical in [0, 2^p - 1)."""
    mp = (1 << p) - 1
    if x < 0:
        x %= mp
    while x > mp:
        x = (x & mp) + (x >> p)
    return 0 if x == mp else x


def lucas_lehmer_steps(p: int, iters: int, s: int = 4) -> int:
    """`iters` device steps s <- (s^2 - 2) mod (2^p - 1) starting from s (0 <= s < 2^p)."""
    plan = _plan_for(max(p, _MIN_PLAN_BITS), word_bits())
    dp = device_plan(plan)
    n = -(-p // 32)
    out = dp.lucas_lehmer(p, iters, int_to_u32(s, n))
    return u32_to_int(out)


def lucas_lehmer(p: int, multiplier: str = "smul", thresholds=None):
    """Lucas-Lehmer test of 2^p - 1 (bigmul/bench.py:197-217) -> (is_prime, residue64).

    Same signature and default multiplier as the reference; an unknown name raises KeyError
    from the table lookup, as the reference's ``ALGORITHMS[multiplier]`` does (bigmul/bench.py:210)."""
    if p == 2:
        return True, 4 & ((1 << 64) - 1)
    if p < 2 or p % 2 == 0:
        raise ValueError("exponent must be an odd prime")
    ALGORITHMS[multiplier]  # KeyError for an unknown rung, before any work
    if multiplier == "smul":
        # the comparison baseline: one GPU smul square per step, reduced on the host
        # (bigmul/bench.py:210-216 with ALGORITHMS["smul"])
        fn = ALGORITHMS["smul"]
        return lucas_lehmer_host(p, square=lambda x: fn(x, x, thresholds, None).to_int())
    if multiplier != "dmul":
        # the reference's other rungs are not part of this build
        ALGORITHMS[multiplier](1, 1, thresholds, None)
    s = lucas_lehmer_steps(p, p - 2, 4)
    return s == 0, s & ((1 << 64) - 1)


def lucas_lehmer_host(p: int, square=None) -> tuple:
    """The same loop with the square supplied by `square` (default: Python ints); used by the
    tests to produce expected residues."""
    if p == 2:
        return True, 4
    s = 4
    for _ in range(p - 2):
        sq = square(s) if square else s * s
        s = mersenne_reduce(sq - 2, p)
    return s == 0, s & ((1 << 64) - 1)


__all__ = ["lucas_lehmer", "lucas_lehmer_host", "lucas_lehmer_steps", "mersenne_reduce"]
