"""Lucas-Lehmer system test (bigmul/bench.py:187-217; tests/test_acceptance.py:219-237 of the
reference): host restatement of mersenne_reduce on CPU, the device loop on the GPU."""
import random

import pytest

from paper_1503_04955_b200.lucas import lucas_lehmer, lucas_lehmer_host, lucas_lehmer_steps, mersenne_reduce

MERSENNE_PRIME_EXPONENTS = (3, 5, 7, 13, 17, 19, 31, 61, 89, 107, 127, 521, 607, 1279, 2203, 2281, 3217, 4253,
                            4423, 9689, 9941, 11213, 19937, 21701, 23209)


def test_mersenne_reduce_matches_mod():
    rng = random.Random(7)
    for p in (3, 31, 61, 89, 127, 521):
        mp = (1 << p) - 1
        for x in [0, 1, mp - 1, mp, mp + 1, 2 * mp, -1, -2, -mp] + [rng.getrandbits(2 * p) for _ in range(20)]:
            assert mersenne_reduce(x, p) == x % mp


def test_host_loop_verdicts():
    for p in (3, 5, 7, 13, 17, 19, 31, 61, 89, 107, 127):
        assert lucas_lehmer_host(p)[0] is True
    for p in (11, 23, 29, 37, 41, 43, 47, 53, 59):
        assert lucas_lehmer_host(p)[0] is False


def test_argument_errors():
    with pytest.raises(ValueError):
        lucas_lehmer(4)
    with pytest.raises(KeyError):  # the reference's ALGORITHMS[multiplier] lookup (bigmul/bench.py:210)
        lucas_lehmer(9, "nope")
    assert lucas_lehmer(2) == (True, 4)
    import inspect

    assert inspect.signature(lucas_lehmer).parameters["multiplier"].default == "smul"  # bigmul/bench.py:197


@pytest.mark.gpu
@pytest.mark.parametrize("p", [3, 5, 7, 11, 13, 23, 29, 31, 37, 61, 89, 127, 521, 1279, 4423])
def test_device_ll_matches_host(cuda_ok, p):
    assert lucas_lehmer(p, "dmul") == lucas_lehmer_host(p)


@pytest.mark.gpu
def test_device_ll_known_primes(cuda_ok):
    for p in MERSENNE_PRIME_EXPONENTS:
        assert lucas_lehmer(p, "dmul")[0] is True, p


@pytest.mark.gpu
def test_device_ll_composite_residues(cuda_ok):
    # residue64 of composite Mersenne numbers against Python's int loop
    for p in (1277, 2311, 4457, 9697, 11239):
        assert lucas_lehmer(p, "dmul") == lucas_lehmer_host(p), p


@pytest.mark.gpu
def test_device_ll_steps_from_random_state(cuda_ok):
    # the device step from arbitrary states, including the edge states 0, 1, 2 and 2^p - 2
    rng = random.Random(3)
    for p in (31, 32 * 40, 32 * 40 + 1, 4423, 65537):
        mp = (1 << p) - 1
        for s in [0, 1, 2, 3, mp - 1, mp - 2, rng.getrandbits(p) % mp]:
            want = s
            for _ in range(3):
                want = mersenne_reduce(want * want - 2, p)
            assert lucas_lehmer_steps(p, 3, s) == want, (p, s)
