"""B200-native DKSS large-integer multiplication (arXiv 1503.04955 hot path).

Drop-in for the reference package's DKSS entry points (bigmul/__init__.py:8-46):
``dmul``, ``mul(..., algorithm="dmul")``, ``ALGORITHMS["dmul"]``,
``dkss_select_params``, ``Natural``, ``ScratchArena``, ``ThresholdTable``.
Parameter selection runs on the host (plan.py); every multiply runs in the
sm_100a kernels of libdkss.so (csrc/), loaded through ctypes (_native.py).
"""

from .dispatch import ALGORITHMS, ThresholdTable, default_thresholds, mul, set_default_thresholds
from .dkss import (dkss_decode, dkss_encode, dkss_fft, dmul, dmul_many, r_mul)
from .lucas import lucas_lehmer, mersenne_reduce
from .plan import DkssPlan, dkss_select_params, make_plan, plan_trace, select_geometry
from .words import Natural, ScratchArena, set_word_bits, using_word_bits, word_bits

__all__ = [
    "ALGORITHMS", "DkssPlan", "Natural", "ScratchArena", "ThresholdTable", "default_thresholds",
    "dkss_decode", "dkss_encode", "dkss_fft", "dkss_select_params", "dmul", "dmul_many", "lucas_lehmer",
    "make_plan", "mersenne_reduce", "mul",
    "plan_trace", "r_mul", "select_geometry", "set_default_thresholds", "set_word_bits", "using_word_bits",
    "word_bits",
]
