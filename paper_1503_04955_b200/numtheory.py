"""Host-side number theory for DKSS plan construction.

Restates the pieces of ``bigmul/numtheory.py`` that plan construction uses
(parameter selection stays in host Python, per BASELINE.json ``north_star``):

* ``modinv``                     -- ``bigmul/numtheory.py:33-48``
* ``factor_smooth``              -- ``bigmul/numtheory.py:51-77`` (trial division)
* ``lucas_prime_test``           -- ``bigmul/numtheory.py:87-107``
* ``find_generator``             -- ``bigmul/numtheory.py:110-120``
* ``find_proth_prime``           -- ``bigmul/numtheory.py:123-143``
* ``is_principal_root``          -- ``bigmul/numtheory.py:175-185``
* ``principal_sums_vanish``      -- ``bigmul/numtheory.py:188-199``
* ``proth_from_record``          -- ``bigmul/numtheory.py:245-246``
* ``proth_table_rows``           -- regenerates the ``bits h g`` records of
  ``bigmul/data/proth_primes.txt`` (rule: ``bigmul/numtheory.py:220-242``).

Python's built-in three-argument ``pow`` is the modular exponentiation
(``bigmul/numtheory.py:17-30`` computes the same function).
"""

from __future__ import annotations

TRIAL_DIVISION_BOUND = 1 << 20


def powmod(base: int, exp: int, modulus: int) -> int:
    if modulus < 2:
        raise ValueError("modulus must be >= 2")
    if exp < 0:
        raise ValueError("negative exponent")
    return pow(base, exp, modulus)


def modinv(x: int, modulus: int) -> int:
    x %= modulus
    a, b, s0, s1 = x, modulus, 1, 0
    while b:
        q = a // b
        a, b = b, a - q * b
        s0, s1 = s1, s0 - q * s1
    if a != 1:
        raise ValueError(f"{x} is not invertible modulo {modulus} (gcd={a})")
    return s0 % modulus


def factor_smooth(n: int):
    """[(prime, exponent), ...] by trial division; odd cofactor must stay small."""
    if n < 1:
        raise ValueError("can only factor positive integers")
    out = []
    twos = (n & -n).bit_length() - 1
    if twos:
        out.append((2, twos))
        n >>= twos
    q = 3
    while q * q <= n and q <= TRIAL_DIVISION_BOUND:
        e = 0
        while n % q == 0:
            n //= q
            e += 1
        if e:
            out.append((q, e))
        q += 2
    if n > 1:
        if n > TRIAL_DIVISION_BOUND * TRIAL_DIVISION_BOUND:
            raise ValueError(f"cofactor {n} exceeds the trial division bound")
        out.append((n, 1))
    return out


def _product(factors) -> int:
    v = 1
    for q, e in factors:
        v *= q ** e
    return v


def lucas_prime_test(n: int, factors) -> bool:
    """Deterministic Lucas test with witnesses a < 1000; ``factors`` factor n-1."""
    if _product(factors) != n - 1:
        raise ValueError("factors do not multiply to n-1")
    if n < 2:
        return False
    if n in (2, 3):
        return True
    if n % 2 == 0:
        return False
    qs = [q for q, _ in factors]
    for a in range(2, 1000):
        if pow(a, n - 1, n) != 1:
            return False
        if all(pow(a, (n - 1) // q, n) != 1 for q in qs):
            return True
    raise ValueError(f"no Lucas witness below 1000 for n={n}")


def find_generator(p: int, p_minus_1_factors=None) -> int:
    """Smallest g >= 2 generating F_p*."""
    if p_minus_1_factors is None:
        p_minus_1_factors = factor_smooth(p - 1)
    qs = [q for q, _ in p_minus_1_factors]
    for g in range(2, p):
        if all(pow(g, (p - 1) // q, p) != 1 for q in qs):
            return g
    raise ValueError(f"no generator found for p={p}")


def _merge(factors):
    acc = {}
    for q, e in factors:
        acc[q] = acc.get(q, 0) + e
    return sorted(acc.items())


def find_proth_prime(two_M: int, min_bits: int):
    """Smallest odd h with p = h*2^k + 1 prime, k = max(log2 2M, min_bits - bitlen h)."""
    if two_M < 2 or two_M & (two_M - 1):
        raise ValueError("two_M must be a power of 2")
    base_k = two_M.bit_length() - 1
    for h in range(1, 1 << 20, 2):
        k = max(base_k, min_bits - h.bit_length())
        p = (h << k) + 1
        factors = _merge([(2, k)] + ([] if h == 1 else factor_smooth(h)))
        try:
            prime = lucas_prime_test(p, factors)
        except ValueError:
            prime = False
        if prime:
            return p, h, find_generator(p, factors)
    raise ValueError(f"no Proth prime for 2M=2^{base_k}, min_bits={min_bits}")


def is_principal_root(omega: int, order: int, p: int) -> bool:
    """For power-of-2 order in a field: omega^(order/2) == -1 and omega^order == 1."""
    if order & (order - 1):
        raise ValueError("order must be a power of 2")
    if order == 1:
        return omega % p == 1
    return pow(omega, order // 2, p) == p - 1 and pow(omega, order, p) == 1


def principal_sums_vanish(omega: int, order: int, modulus: int) -> bool:
    for j in range(1, order):
        wj = pow(omega, j, modulus)
        acc, x = 0, 1
        for _ in range(order):
            acc = (acc + x) % modulus
            x = x * wj % modulus
        if acc:
            return False
    return True


def proth_from_record(bits: int, h: int) -> int:
    return (h << (bits - h.bit_length())) + 1


def proth_record(bits: int, min_two_m: int = 64):
    """One ``(bits, h, g)`` record of the planner's prime table."""
    two_m = min(min_two_m, 1 << max(1, bits - 2))
    p, h, g = find_proth_prime(two_m, bits)
    if p.bit_length() != bits:
        raise ValueError(f"search returned {p.bit_length()}-bit prime for bits={bits}")
    return bits, h, g


def proth_table_rows(max_bits: int = 1704, step: int = 8, min_two_m: int = 64):
    return [proth_record(bits, min_two_m) for bits in range(step, max_bits + 1, step)]
