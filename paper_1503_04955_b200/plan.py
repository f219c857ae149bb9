"""DKSS parameter selection and root construction (host side, Python).

BASELINE.json ``north_star``: "The parameter selection (M, m, u, p, c, rho)
stays in host Python, exactly as in the reference."  This module restates the
reference's planner so that every field of the plan equals the reference's
(pinned by tests/test_plan_golden.py against golden values produced by the
reference itself, see tools/make_golden.py):

* ``DkssPlan``            -- ``bigmul/dkss.py:97-146`` (fields, derived sizes,
                              ``validate_sizes``)
* ``find_root_omega``     -- ``bigmul/dkss.py:152-157``
* ``compute_rho``         -- ``bigmul/dkss.py:160-195`` (Lagrange interpolation
                              of rho through (gamma^i, omega^i), i odd)
* ``make_plan``           -- ``bigmul/dkss.py:207-240`` (rho-power cache keyed
                              by (p, M, m))
* ``verify_rho``          -- ``bigmul/dkss.py:257-269``
* ``proth_table`` / ``proth_for_bits`` -- ``bigmul/dkss.py:286-308``
* ``select_geometry``     -- ``bigmul/dkss.py:314-352``
* ``dkss_select_params``  -- ``bigmul/dkss.py:355-361``
* ``plan_trace``          -- ``bigmul/dkss.py:364-375``

On top of the reference fields the plan carries the *device layout* the GPU
path needs (limb count L, level structure of the radix-2m transform); those
are derived, never chosen.
"""

from __future__ import annotations

import math
import os
import threading
from dataclasses import dataclass, field

from .numtheory import factor_smooth, find_generator, is_principal_root, modinv, proth_from_record
from .words import word_bits


# ---------------------------------------------------------------------------
# small exact ring helpers on coefficient lists (host only: root setup + tests)

def poly_mul_mod(x, y, m: int, p: int):
    """Schoolbook product in P[alpha]/(alpha^m+1) (``bigmul/dkss.py:243-254``)."""
    acc = [0] * (2 * m)
    for i, xi in enumerate(x):
        if xi:
            for j, yj in enumerate(y):
                acc[i + j] += xi * yj
    return [(acc[k] - acc[k + m]) % p for k in range(m)]


def poly_pow(x, e: int, m: int, p: int):
    out = [1] + [0] * (m - 1)
    base = list(x)
    while e:
        if e & 1:
            out = poly_mul_mod(out, base, m, p)
        base = poly_mul_mod(base, base, m, p)
        e >>= 1
    return out


def poly_mul_xpow(x, e: int, m: int, p: int):
    """x * alpha^e: rotate by e, negating wrapped coefficients (``bigmul/dkss.py:46-61``)."""
    e %= 2 * m
    out = [0] * m
    for i, c in enumerate(x):
        j = i + e
        neg = False
        while j >= m:
            j -= m
            neg = not neg
        out[j] = (p - c if c else 0) if neg else c
    return out


# ---------------------------------------------------------------------------
# the plan

@dataclass
class DkssPlan:
    N: int
    M: int
    m: int
    u: int
    p: int
    z: int
    d: int
    zeta: int
    omega: int
    gamma: int
    rho: list
    rho_powers: list
    w: int
    ks_calls: int = 0

    @property
    def mu(self) -> int:
        return self.M // self.m

    @property
    def pz(self) -> int:
        return self.p ** self.z

    @property
    def iclen(self) -> int:
        return -(-self.d // self.w)

    @property
    def oclen(self) -> int:
        return self.m * self.iclen

    @property
    def ks_stride(self) -> int:
        return 2 * self.d + (self.m.bit_length() - 1)

    # -- device layout (derived) -------------------------------------------
    @property
    def L(self) -> int:
        """u32 limbs per residue on the device."""
        return -(-self.d // 32)

    @property
    def levels(self) -> int:
        """Number of radix-2m column passes before the base case."""
        n, k = 2 * self.M, 0
        while n > 2 * self.m:
            n //= 2 * self.m
            k += 1
        return k

    @property
    def base_len(self) -> int:
        return (2 * self.M) // (2 * self.m) ** self.levels

    def validate_sizes(self) -> "DkssPlan":
        if self.m < 2 or self.M < self.m:
            raise ValueError("need M >= m >= 2")
        if self.M & (self.M - 1) or self.m & (self.m - 1):
            raise ValueError("M and m must be powers of 2")
        if self.u != -(-2 * self.N // (self.M * self.m)):
            raise ValueError("u must equal ceil(2N / Mm)")
        if self.pz < (self.M * self.m) << (2 * self.u):
            raise ValueError("p^z below the coefficient bound Mm*2^(2u)")
        if (self.p - 1) % (2 * self.M):
            raise ValueError("2M must divide p-1")
        return self


_cache_lock = threading.Lock()
_rho_cache: dict = {}


def find_root_omega(p: int, two_M: int, zeta: int) -> int:
    omega = pow(zeta, (p - 1) // two_M, p)
    if not is_principal_root(omega, two_M, p):
        raise ValueError(f"zeta={zeta} does not yield a principal 2M-th root mod {p}")
    return omega


def _times_linear(poly, root: int, p: int):
    """poly(alpha) * (alpha - root)."""
    out = [0] * (len(poly) + 1)
    for i, c in enumerate(poly):
        out[i + 1] = (out[i + 1] + c) % p
        out[i] = (out[i] - c * root) % p
    return out


def compute_rho(p: int, M: int, m: int, omega: int):
    """rho in R with rho == omega^i mod (alpha - gamma^i) for every odd i < 2m.

    gamma = omega^(M/m) has order 2m, so its odd powers are the m roots of
    alpha^m + 1; interpolating rho through (gamma^i, omega^i) gives
    rho^(M/m) = alpha and rho^(2M) = 1 (``PAPER.md:2235-2238``).
    """
    gamma = pow(omega, M // m, p)
    odd = range(1, 2 * m, 2)
    g = {i: pow(gamma, i, p) for i in odd}
    prod = [1]
    for i in odd:
        prod = _times_linear(prod, g[i], p)
    if [c % p for c in prod] != [1] + [0] * (m - 1) + [1]:
        raise ValueError("gamma powers do not factor alpha^m + 1")
    rho = [0] * m
    for i in odd:
        gi = g[i]
        # (alpha^m + 1) / (alpha - gi): coefficient j is gi^(m-1-j)
        quot = [pow(gi, m - 1 - j, p) for j in range(m)]
        den = 1
        for j in odd:
            if j != i:
                den = den * (gi - g[j]) % p
        scale = pow(omega, i, p) * modinv(den, p) % p
        for j in range(m):
            rho[j] = (rho[j] + quot[j] * scale) % p
    return rho, gamma


def verify_rho(plan: DkssPlan) -> None:
    q = poly_pow(plan.rho, plan.mu, plan.m, plan.p)
    alpha = [0, 1] + [0] * (plan.m - 2) if plan.m > 1 else [plan.p - 1]
    if q != alpha:
        raise ValueError("rho^(2M/2m) != alpha")
    r = q
    for _ in range(plan.m.bit_length()):
        r = poly_mul_mod(r, r, plan.m, plan.p)
    if r != [1] + [0] * (plan.m - 1):
        raise ValueError("rho^(2M) != 1")


def make_plan(N: int, M: int, m: int, p: int, zeta: int | None = None,
              w: int | None = None, check_bounds: bool = True) -> DkssPlan:
    w = word_bits() if w is None else w
    if zeta is None:
        zeta = find_generator(p, factor_smooth(p - 1))
    u = -(-2 * N // (M * m)) if N else 0
    key = (p, M, m)
    with _cache_lock:
        hit = _rho_cache.get(key)
    if hit is None:
        omega = find_root_omega(p, 2 * M, zeta)
        rho, gamma = compute_rho(p, M, m, omega)
        mu = M // m
        powers = [[1] + [0] * (m - 1)]
        for _ in range(1, mu):
            powers.append(poly_mul_mod(powers[-1], rho, m, p))
        hit = (omega, gamma, rho, powers)
        with _cache_lock:
            _rho_cache.setdefault(key, hit)
    omega, gamma, rho, powers = hit
    plan = DkssPlan(N, M, m, u, p, 1, p.bit_length(), zeta, omega, gamma, rho, powers, w)
    if check_bounds:
        plan.validate_sizes()
    verify_rho(plan)
    return plan


# ---------------------------------------------------------------------------
# prime table

_table_lock = threading.Lock()
_PROTH_ROWS: dict | None = None


def proth_table() -> dict:
    global _PROTH_ROWS
    with _table_lock:
        if _PROTH_ROWS is None:
            path = os.path.join(os.path.dirname(__file__), "data", "proth_primes.txt")
            rows = {}
            with open(path) as f:
                for line in f:
                    line = line.split("#", 1)[0].strip()
                    if line:
                        bits, h, g = map(int, line.split())
                        rows[bits] = (proth_from_record(bits, h), h, g)
            _PROTH_ROWS = rows
        return _PROTH_ROWS


def proth_for_bits(bits: int):
    rows = proth_table()
    if bits not in rows:
        raise ValueError(f"no precomputed Proth prime with {bits} bits")
    return rows[bits]


# ---------------------------------------------------------------------------
# parameter selection

def select_geometry(N: int, w: int | None = None):
    """(M, m, u, p, generator) for inputs below 2^N (``bigmul/dkss.py:314-352``).

    Prime width first: ceil(5 log N - 1 - log log N) rounded up to a word
    multiple; then the smallest power-of-2 Mm with Mm * 2^(2u) <= p,
    u = ceil(2N/Mm); then m (power of 2, m^2 <= Mm) closest in log scale to
    Mm/m^2 ~ N / log^3 N.
    """
    w = word_bits() if w is None else w
    if N < 32:
        raise ValueError("input too small for a DKSS plan")
    lg = math.log2(N)
    d_target = max(1, math.ceil(5 * lg - 1 - math.log2(lg)))
    d = -(-d_target // w) * w
    p, _h, g = proth_for_bits(d)
    mm = 4
    while True:
        u = -(-2 * N // mm)
        if u >= 1 and mm << (2 * u) <= p:
            break
        mm <<= 1
        if mm > 2 * N:
            raise ValueError(f"no feasible Mm for N={N} with a {d}-bit prime")
    target = N / lg ** 3
    best = None
    cand = 2
    while cand * cand <= mm:
        dist = abs(math.log2((mm / (cand * cand)) / target))
        if best is None or dist < best[1]:
            best = (cand, dist)
        cand <<= 1
    m = best[0]
    M = mm // m
    if (p - 1) % (2 * M):
        raise ValueError(f"table prime {p} lacks 2-adic room for 2M={2 * M}")
    return M, m, u, p, g


def dkss_select_params(N: int, w: int | None = None, table=None) -> DkssPlan:
    w = word_bits() if w is None else w
    M, m, u, p, g = select_geometry(N, w)
    return make_plan(N, M, m, p, zeta=g, w=w)


def plan_trace(plan: DkssPlan) -> str:
    return "\n".join([
        f"N={plan.N} bits  M={plan.M}  m={plan.m}  mu={plan.mu}  u={plan.u}",
        f"p={plan.p} ({plan.d} bits, z={plan.z})  zeta={plan.zeta}",
        f"omega={plan.omega}  gamma={plan.gamma}",
        f"inner residue: {plan.iclen} words; outer coefficient: {plan.oclen} words",
        f"kronecker stride: {plan.ks_stride} bits -> packed {plan.m * plan.ks_stride} bits",
        f"fft vector: {2 * plan.M} outer coefficients, "
        f"{2 * plan.M * plan.oclen * plan.w // 8} bytes each polynomial",
        f"device: L={plan.L} u32 limbs/residue, {plan.levels} radix-{2 * plan.m} column passes, "
        f"base length {plan.base_len}",
    ])


def twiddle_count(plan: DkssPlan) -> int:
    """Ring products one dkss_fft performs (what ``plan.ks_calls`` counts per FFT)."""
    def rec(length: int) -> int:
        if length <= 2 * plan.m:
            return 0
        mu = length // (2 * plan.m)
        return (2 * plan.m - 1) * (mu - 1) + 2 * plan.m * rec(mu)
    return rec(2 * plan.M)


def ring_products_per_multiply(plan: DkssPlan) -> int:
    """3 transforms + 2M pointwise products."""
    return 3 * twiddle_count(plan) + 2 * plan.M
