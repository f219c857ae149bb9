"""Host-side number representation shared with the reference multiply API.

The reference passes operands as Python ints or as ``Natural`` (little-endian
w-bit word lists, w thread-local, default 64; ``bigmul/words.py:17-41``,
``bigmul/words.py:56-117``).  This module restates exactly the parts of that
contract the DKSS entry points touch:

* ``Natural`` construction / ``to_int`` / ``len`` / equality semantics
  (``bigmul/words.py:56-109``) -- needed because ``dmul`` returns a Natural of
  exactly ``len(a) + len(b)`` words (``bigmul/dkss.py:529,548``);
* ``as_natural`` type checks (``bigmul/words.py:112-117``);
* thread-local word size (``bigmul/words.py:17-41``) -- the DKSS plan depends
  on it (d is rounded to a multiple of w, ``bigmul/dkss.py:327-328``);
* ``ScratchArena`` accounting (``bigmul/words.py:234-304``) -- accepted by the
  API; the GPU path records its device workspace in it;
* ``bit_slices`` / ``join_bits`` (``bigmul/words.py:307-349``) -- the encode /
  decode semantics, used here only by host-side helpers and tests.

Conversion between ints and the u32 limb arrays that cross the C ABI is done
with ``int.to_bytes`` / ``numpy.frombuffer`` (no per-word Python loops).
"""

from __future__ import annotations

import ctypes
import sys
import threading
from contextlib import contextmanager

import numpy as np

_WORD_SIZES = (8, 16, 32, 64)
_tls = threading.local()


def word_bits() -> int:
    return getattr(_tls, "w", 64)


def word_base() -> int:
    return 1 << word_bits()


def set_word_bits(w: int) -> None:
    if w not in _WORD_SIZES:
        raise ValueError(f"unsupported word size {w}, pick one of {_WORD_SIZES}")
    _tls.w = w


@contextmanager
def using_word_bits(w: int):
    prev = word_bits()
    set_word_bits(w)
    try:
        yield
    finally:
        set_word_bits(prev)


def _words_needed(value: int, w: int) -> int:
    return max(1, -(-value.bit_length() // w))


def int_to_words(value: int, length: int, w: int) -> list:
    if length == 0:
        return []
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[w]
    raw = value.to_bytes(length * (w // 8), "little")
    return np.frombuffer(raw, dtype=dt).tolist()


def words_to_int(words, w: int) -> int:
    if len(words) == 0:
        return 0
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[w]
    return int.from_bytes(np.asarray(words, dtype=dt).tobytes(), "little")


class Natural:
    """Nonnegative integer as little-endian words of the current word size.

    Mirrors ``bigmul.words.Natural``: leading zero words are allowed, the
    object is treated as immutable, equality compares values (also against
    plain ints).  Products coming back from the device keep their limb array
    and build the word list only when ``words`` is first read.
    """

    __slots__ = ("_words", "_limbs", "_w", "_len", "_ival", "_iw")

    def __init__(self, words):
        self._words = list(words)
        self._limbs = None
        self._w = None
        self._len = len(self._words)
        self._ival = None  # value cache (the object is immutable): (value, word size it was read at)
        self._iw = None

    @classmethod
    def _from_u32(cls, limbs: np.ndarray, length: int, w: int) -> "Natural":
        """Natural of `length` w-bit words from little-endian u32 limbs (no per-word Python work)."""
        obj = cls.__new__(cls)
        need = -(-length * w // 32)
        if limbs.size < need:
            limbs = np.concatenate([limbs, np.zeros(need - limbs.size, dtype=np.uint32)])
        obj._limbs = limbs[:need] if (length * w) % 32 == 0 else limbs
        obj._w = w
        obj._len = length
        obj._words = None
        obj._ival = None
        obj._iw = None
        return obj

    @property
    def words(self) -> list:
        if self._words is None:
            dt = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[self._w]
            raw = np.ascontiguousarray(self._limbs, dtype=np.uint32).tobytes()
            nbytes = self._len * self._w // 8
            raw = raw[:nbytes] + b"\0" * max(0, nbytes - len(raw))
            self._words = np.frombuffer(raw, dtype=dt).tolist()
            self._limbs = None
        return self._words

    @classmethod
    def from_int(cls, value: int, length: int | None = None, w: int | None = None) -> "Natural":
        if value < 0:
            raise ValueError("Natural is nonnegative")
        w = word_bits() if w is None else w
        need = _words_needed(value, w)
        if length is None:
            length = need
        elif length < need:
            raise ValueError(f"value needs {need} words, got length={length}")
        obj = cls(int_to_words(value, length, w))
        obj._ival, obj._iw = value, w
        return obj

    def to_int(self, w: int | None = None) -> int:
        w = word_bits() if w is None else w
        if self._iw == w:
            return self._ival
        if self._words is None and w == self._w:
            v = int.from_bytes(np.ascontiguousarray(self._limbs, dtype=np.uint32).tobytes(), "little")
        else:
            v = words_to_int(self.words, w)
        self._ival, self._iw = v, w
        return v

    def normalized(self) -> "Natural":
        ws = self.words
        n = len(ws)
        while n > 1 and ws[n - 1] == 0:
            n -= 1
        return Natural(ws[:n])

    def bit_length(self, w: int | None = None) -> int:
        return self.to_int(w).bit_length()

    def __len__(self) -> int:
        return self._len

    def __eq__(self, other) -> bool:
        if isinstance(other, Natural):
            return self.to_int() == other.to_int()
        if isinstance(other, int):
            return self.to_int() == other
        fw = foreign_natural(other)
        if fw is not None:  # the reference's bigmul.words.Natural (or any word-list Natural)
            return self.to_int() == words_to_int(other.words, fw[1])
        return NotImplemented

    __hash__ = None

    def __repr__(self) -> str:
        return f"Natural({self.words!r})"


def foreign_natural(x):
    """(class, word size) when x is another package's Natural -- an object with a ``words`` list
    and ``to_int``, like the reference's ``bigmul.words.Natural`` (bigmul/words.py:56-109) -- else
    None.  Its words are at ITS package's thread-local word size: the reference keeps its own
    ``word_bits()`` (bigmul/words.py:17-23), read from the class's module when it has one."""
    if isinstance(x, (Natural, int)) or not hasattr(x, "words") or not hasattr(x, "to_int"):
        return None
    mod = sys.modules.get(type(x).__module__)
    wb = getattr(mod, "word_bits", None)
    w = wb() if callable(wb) else word_bits()
    return type(x), w


def as_natural(x) -> Natural:
    if isinstance(x, Natural):
        return x
    fw = foreign_natural(x)
    if fw is not None:  # same words at the same word size; else the same value
        return Natural(x.words) if fw[1] == word_bits() else Natural.from_int(words_to_int(x.words, fw[1]))
    if isinstance(x, int) and not isinstance(x, bool):
        return Natural.from_int(x)
    if isinstance(x, bool):
        return Natural.from_int(int(x))
    raise TypeError(f"expected int or Natural, got {type(x).__name__}")


class ScratchArena:
    """LIFO scratch accounting in machine words (``bigmul/words.py:234-286``).

    The GPU path allocates its workspace once per plan; it still reports the
    words it keeps live per multiply through ``alloc_words`` so the arena's
    ``peak_words`` remains a meaningful memory instrument.
    """

    __slots__ = ("pos", "peak_words", "reserved_words")

    def __init__(self):
        self.pos = 0
        self.peak_words = 0
        self.reserved_words = 0

    def acquire(self) -> int:
        return self.pos

    def release(self, mark: int) -> None:
        if not 0 <= mark <= self.pos:
            raise ValueError("release does not match an acquire mark")
        self.pos = mark
        self.reserved_words = max(self.reserved_words, self.peak_words)

    @contextmanager
    def frame(self):
        mark = self.acquire()
        try:
            yield self
        finally:
            self.release(mark)

    def alloc_words(self, nwords: int) -> None:
        if nwords < 0:
            raise ValueError("negative allocation")
        self.pos += nwords
        self.peak_words = max(self.peak_words, self.pos)

    def alloc_list(self, count: int, words_per_item: int, fill=0) -> list:
        self.alloc_words(count * words_per_item)
        return [fill] * count

    def reset_stats(self) -> None:
        self.peak_words = 0

    def peak_bytes(self, w: int | None = None) -> int:
        return self.peak_words * ((word_bits() if w is None else w) // 8)


def current_arena() -> ScratchArena:
    arena = getattr(_tls, "arena", None)
    if arena is None:
        arena = _tls.arena = ScratchArena()
    return arena


@contextmanager
def use_arena(arena: ScratchArena):
    prev = getattr(_tls, "arena", None)
    _tls.arena = arena
    try:
        yield arena
    finally:
        _tls.arena = prev


def bit_slices(value: int, width: int, count: int) -> list:
    """``count`` little-endian fields of ``width`` bits (``bigmul/words.py:307-329``)."""
    if width <= 0:
        raise ValueError("field width must be positive")
    mask = (1 << width) - 1
    return [(value >> (i * width)) & mask for i in range(count)]


def join_bits(parts, width: int) -> int:
    """sum(parts[i] << width*i); parts may exceed ``width`` (``bigmul/words.py:332-349``)."""
    # pairwise tree combination keeps this O(n log n) for long part lists
    vals = [int(p) for p in parts]
    shift = width
    while len(vals) > 1:
        nxt = [vals[i] + (vals[i + 1] << shift) for i in range(0, len(vals) - 1, 2)]
        if len(vals) & 1:
            nxt.append(vals[-1])
        vals = nxt
        shift *= 2
    return vals[0] if vals else 0


# ---------------------------------------------------------------------------
# int <-> u32 limb arrays for the C ABI

def int_to_u32(value: int, nlimbs: int) -> np.ndarray:
    """Little-endian uint32 limbs, zero-padded to ``nlimbs``."""
    if value < 0:
        raise ValueError("negative operand")
    return np.frombuffer(value.to_bytes(4 * nlimbs, "little"), dtype=np.uint32).copy()


def u32_to_int(limbs) -> int:
    return int.from_bytes(np.ascontiguousarray(limbs, dtype=np.uint32).tobytes(), "little")


# ---------------------------------------------------------------------------
# zero-copy view of a CPython int's digits (CPython >= 3.12 object layout: PyObject header,
# then uintptr lv_tag = ndigits << 3 | sign, then the 30-bit digits, one per uint32).  The
# multiply hands these digits to the C ABI as they are (dkss_mul_digits) instead of
# converting the int with to_bytes, which is a byte-at-a-time loop in CPython.

def _raw_digits(x: int):
    tag = ctypes.c_size_t.from_address(id(x) + 16).value
    return id(x) + 24, tag >> 3, tag & 3


def _layout_ok() -> bool:
    if sys.implementation.name != "cpython" or sys.version_info < (3, 12):
        return False
    if sys.int_info.bits_per_digit != 30 or sys.int_info.sizeof_digit != 4:
        return False
    try:
        x = (7 << 60) | (3 << 30) | 5
        addr, nd, sign = _raw_digits(x)
        if (nd, sign) != (3, 0) or list((ctypes.c_uint32 * 3).from_address(addr)) != [5, 3, 7]:
            return False
        addr, nd, sign = _raw_digits(-x)
        return (nd, sign) == (3, 2)
    except Exception:  # noqa: BLE001
        return False


PYLONG_DIGIT_BITS = 30
_PYLONG_OK = _layout_ok()


def pylong_digits(x: int):
    """(address, digit count) of the 30-bit digits of a nonnegative int, or None when the
    interpreter's int layout is not the one checked above.  The int must stay alive while
    the address is used.  (The count of a normalised int is ceil(bit_length / 30); the
    digits start at a fixed offset -- both checked against the object header at import.)"""
    if not _PYLONG_OK or type(x) is not int:
        return None
    if x < 0:
        raise ValueError("Natural is nonnegative")
    return id(x) + 24, (x.bit_length() + 29) // 30
