"""Benchmark harness restated from bigmul/bench.py:16-108 (host logic on CPU, dmul on GPU)."""
import io

import pytest

from paper_1503_04955_b200 import harness
from paper_1503_04955_b200.harness import BenchRecord, quotient_column, run_bench, write_csv


def test_csv_and_quotient():
    recs = [BenchRecord("dmul", 1024, 3, 300, 10), BenchRecord("smul", 1024, 3, 100, 5),
            BenchRecord("dmul", 2048, 3, 500, 20)]
    out = io.StringIO()
    write_csv(recs, out)
    lines = out.getvalue().splitlines()
    assert lines[0] == "algorithm,input_words,reps,median_ns,peak_arena_words"
    assert lines[1] == "dmul,1024,3,300,10" and len(lines) == 4
    assert quotient_column(recs) == [(1024, 3.0)]


def test_validation_and_grid():
    with pytest.raises(ValueError):
        run_bench(["dmul"], [2, 1])
    with pytest.raises(ValueError):
        run_bench(["dmul"], [1], reps=2)
    g = harness.default_size_grid(1 << 13)
    assert g == sorted(set(g)) and 1 in g and 8192 in g and 3648 in g and 14336 not in g


def test_timed_products_are_checked(monkeypatch):
    # an algorithm that returns a wrong product must raise, never produce a record
    from paper_1503_04955_b200 import dispatch
    from paper_1503_04955_b200.words import Natural

    monkeypatch.setitem(dispatch.ALGORITHMS, "broken", lambda a, b, t, ar: Natural.from_int(a.to_int() * b.to_int() + 1))
    with pytest.raises(harness.BenchCorrectnessError):
        run_bench(["broken"], [4], reps=3)
    monkeypatch.setitem(dispatch.ALGORITHMS, "exact", lambda a, b, t, ar: Natural.from_int(a.to_int() * b.to_int()))
    recs = run_bench(["exact"], [4, 8], reps=3, seed=1)
    assert [(r.algorithm, r.input_words, r.reps) for r in recs] == [("exact", 4, 3), ("exact", 8, 3)]


@pytest.mark.gpu
def test_run_bench_dmul(cuda_ok):
    recs = run_bench(["dmul"], [64, 1024, 16384], reps=3, seed=5)
    assert [r.input_words for r in recs] == [64, 1024, 16384] and all(r.median_ns > 0 for r in recs)
    assert all(r.peak_arena_words > 0 for r in recs)
