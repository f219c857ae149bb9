"""Boundary types mirror bigmul/words.py (Natural, as_natural, bit_slices/join_bits, arena)."""
import random

import numpy as np
import pytest

from paper_1503_04955_b200.words import (Natural, ScratchArena, as_natural, bit_slices, int_to_u32, join_bits,
                                         u32_to_int, using_word_bits, word_bits)


def test_natural_roundtrip_and_length():
    v = (1 << 200) + 12345
    n = Natural.from_int(v)
    assert n.to_int() == v and len(n) == 4 and n == v
    assert len(Natural.from_int(v, length=10)) == 10
    with pytest.raises(ValueError):
        Natural.from_int(v, length=2)
    with pytest.raises(ValueError):
        Natural.from_int(-1)
    assert Natural([5, 0, 0]).normalized().words == [5]


def test_word_size_thread_local_semantics():
    assert word_bits() == 64
    with using_word_bits(8):
        n = Natural.from_int(0x1234)
        assert n.words == [0x34, 0x12]
    assert word_bits() == 64


def test_as_natural_types():
    assert as_natural(7) == 7
    with pytest.raises(TypeError):
        as_natural(1.5)
    with pytest.raises(ValueError):
        as_natural(-3)


def test_bit_slices_join_bits(rng):
    for width in (13, 32, 79):
        v = rng.getrandbits(width * 20)
        parts = bit_slices(v, width, 20)
        assert join_bits(parts, width) == v
    # parts wider than the stride overlap and add (bigmul/words.py:332-349)
    assert join_bits([3, 5], 1) == 3 + 10


def test_u32_limbs(rng):
    v = rng.getrandbits(1000)
    limbs = int_to_u32(v, 40)
    assert limbs.dtype == np.uint32 and limbs.size == 40 and u32_to_int(limbs) == v


def test_scratch_arena_peak():
    a = ScratchArena()
    with a.frame():
        a.alloc_words(10)
        with a.frame():
            a.alloc_words(5)
        a.alloc_words(1)
    assert a.pos == 0 and a.peak_words == 15


def test_pylong_digits_layout_and_fallback(monkeypatch):
    # e2e hands CPython's own 30-bit int digits to the C ABI (words.pylong_digits, checked
    # against the interpreter's int layout at import); without that layout (another
    # interpreter, a layout change) the operand goes as 32-bit limbs instead -- same product
    import ctypes

    import numpy as np

    from paper_1503_04955_b200 import dkss, words

    x = (1 << 1000) + 12345678901234567890
    d = words.pylong_digits(x)
    if d is not None:  # CPython >= 3.12: the digits read back are the int's base-2^30 digits
        ptr, n = d
        got = np.ctypeslib.as_array((ctypes.c_uint32 * n).from_address(ptr)).copy()
        want = [(x >> (30 * i)) & ((1 << 30) - 1) for i in range(n)]
        assert got.tolist() == want
        keep, p, cnt, bits = dkss._digits(x, x)
        assert (p, cnt) == (ptr, n) and bits & 0xFF == words.PYLONG_DIGIT_BITS
    monkeypatch.setattr(words, "_PYLONG_OK", False)
    assert words.pylong_digits(x) is None
    keep, p, cnt, bits = dkss._digits(x, x)
    assert bits == 32 and np.array_equal(keep, words.int_to_u32(x, cnt))
