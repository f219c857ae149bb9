"""Benchmark harness for the GPU dmul rung.

Restates the reference harness (bigmul/bench.py:16-108): ``run_bench`` times every
(algorithm, size) pair ``reps`` times, checks every timed product bit-exactly before it is
reported, and keeps the median; ``write_csv`` / ``quotient_column`` produce the CSV and the
T_num/T_den column of the thesis's run-time table.  The ``"dmul"`` and ``"smul"`` rungs run
on the GPU, so ``quotient_column(records)`` is the thesis's T_DMUL / T_SMUL; the default
check is Python's own int product (``reference=None``); naming another rung raises
NotImplementedError through ALGORITHMS, as ``mul`` does.
"""

from __future__ import annotations

import random
import statistics
import time
from dataclasses import dataclass

from .dispatch import ALGORITHMS, ThresholdTable, default_thresholds
from .words import Natural, ScratchArena, word_bits


class BenchCorrectnessError(RuntimeError):
    """A timed product disagreed with the reference product (bigmul/bench.py:16-17)."""


@dataclass
class BenchRecord:
    algorithm: str
    input_words: int
    reps: int
    median_ns: int
    peak_arena_words: int

    CSV_HEADER = "algorithm,input_words,reps,median_ns,peak_arena_words"

    def csv_row(self) -> str:
        return f"{self.algorithm},{self.input_words},{self.reps},{self.median_ns},{self.peak_arena_words}"


def random_operand(rng: random.Random, words: int) -> Natural:
    """`words` random words with the top word live (bigmul/bench.py:35-39)."""
    bits = words * word_bits()
    return Natural.from_int(rng.getrandbits(bits) | (1 << (bits - 1)), length=words)


def run_bench(algorithms, sizes, reps: int = 3, seed: int = 0, reference: str | None = None,
              thresholds: ThresholdTable | None = None):
    """One BenchRecord per (algorithm, size), each timed product checked first
    (bigmul/bench.py:42-71); reference=None checks against Python's int product."""
    sizes = list(sizes)
    if sizes != sorted(sizes):
        raise ValueError("sizes must be ascending")
    if reps < 3:
        raise ValueError("reps must be at least 3, records hold a median")
    table = thresholds or default_thresholds()
    rng = random.Random(seed)
    records = []
    for size in sizes:
        a, b = random_operand(rng, size), random_operand(rng, size)
        if reference is None:
            ref = a.to_int() * b.to_int()
        else:
            ref = ALGORITHMS[reference](a, b, table, ScratchArena()).to_int()
        for name in algorithms:
            fn = ALGORITHMS[name]
            arena = ScratchArena()
            times = []
            for _ in range(reps):
                t0 = time.perf_counter_ns()
                out = fn(a, b, table, arena)
                times.append(time.perf_counter_ns() - t0)
                if out.to_int() != ref:
                    raise BenchCorrectnessError(f"{name} disagrees with {reference or 'int'} at {size} words")
            records.append(BenchRecord(name, size, reps, int(statistics.median(times)), arena.peak_words))
    return records


def write_csv(records, stream) -> None:
    stream.write(BenchRecord.CSV_HEADER + "\n")
    for rec in records:
        stream.write(rec.csv_row() + "\n")


def quotient_column(records, num: str = "dmul", den: str = "smul"):
    """[(words, T_num / T_den)] for the sizes both algorithms ran (bigmul/bench.py:80-91)."""
    by_size: dict = {}
    for rec in records:
        by_size.setdefault(rec.input_words, {})[rec.algorithm] = rec.median_ns
    return [(size, row[num] / row[den]) for size, row in sorted(by_size.items())
            if num in row and den in row and row[den]]


# the DKSS-favourable lengths of the thesis's run-time table (bigmul/bench.py:94-96)
FAVORABLE_WORDS = [3648, 7168, 14336, 28160, 56320, 110592, 221184]


def default_size_grid(max_words: int = 1 << 14):
    """Powers of two up to max_words plus the favourable lengths (bigmul/bench.py:99-107)."""
    sizes = {1 << k for k in range(max_words.bit_length()) if 1 << k <= max_words}
    sizes.update(s for s in FAVORABLE_WORDS if s <= max_words)
    return sorted(sizes)
