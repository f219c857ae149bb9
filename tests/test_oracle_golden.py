"""Pin the CPU oracle (oracle/dkss_oracle.c, a C restatement of bigmul/dkss.py) on vectors
the reference produced: every stage of 7 real plans, r_mul at the config prime, toy-plan
transforms from the reference's own tests.  CPU only."""
import json
import os
import random
import types

import numpy as np
import pytest

from oracle.oracle import OraclePlan
from paper_1503_04955_b200 import plan as P
from paper_1503_04955_b200.words import u32_to_int, using_word_bits


def _stage_tags(golden_dir):
    with open(os.path.join(golden_dir, "stages_index.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("idx", range(7))
def test_oracle_stages_equal_reference(golden_dir, idx):
    r = _stage_tags(golden_dir)[idx]
    g = np.load(os.path.join(golden_dir, f"stages_{r['tag']}.npz"))
    with using_word_bits(r["w"]):
        pl = P.dkss_select_params(r["N"], r["w"])
    o = OraclePlan(pl)
    a, b = u32_to_int(g["a"]), u32_to_int(g["b"])
    assert np.array_equal(o.encode(a), g["enc_a"])
    assert np.array_equal(o.encode(b), g["enc_b"])
    o.ks_calls(reset=True)
    assert np.array_equal(o.fft(g["enc_a"]), g["fft_a"])
    assert o.ks_calls(reset=True) == r["fft_calls"]        # bigmul/dkss.py:412 instrumentation
    assert np.array_equal(o.fft(g["enc_b"]), g["fft_b"])
    assert np.array_equal(o.rmul(g["fft_a"], g["fft_b"]), g["pointwise"])
    assert np.array_equal(o.fft(g["pointwise"]), g["fft_c"])
    assert np.array_equal(o.decode(g["fft_c"], g["product"].size), g["product"])
    assert o.dmul(a, b) == a * b


@pytest.mark.parametrize("tag", ["m16", "m32"])
def test_oracle_rmul_equal_reference(golden_dir, tag):
    g = np.load(os.path.join(golden_dir, f"rmul_{tag}.npz"))
    m = g["x"].shape[1]
    pl = P.make_plan(0, m, m, u32_to_int(g["p"]), check_bounds=False)
    assert np.array_equal(OraclePlan(pl).rmul(g["x"], g["y"]), g["z"])


def _toy_oracle(t):
    pl = types.SimpleNamespace(N=0, M=t["M"], m=t["m"], u=0, p=t["p"], rho_powers=t["rho_powers"])
    return OraclePlan(pl)


def test_oracle_toy_plans_equal_reference(golden_dir):
    with open(os.path.join(golden_dir, "ref_tests.json")) as f:
        ref = json.load(f)
    for t in ref["toy_plans"]:
        o = _toy_oracle(t)
        arr = lambda v: np.array(v, dtype=np.uint32).reshape(len(v), t["m"], 1)  # noqa: E731
        assert np.array_equal(o.fft(arr(t["fft_in"])), arr(t["fft_out"]))   # tests/test_dkss.py:185-202
        assert np.array_equal(o.rmul(arr(t["x"]), arr(t["y"])), arr(t["z"]))  # tests/test_dkss.py:111-119
    # the first toy plan has 2M == 2m: the whole transform is one inner DFT (the reference's
    # bottom case, tests/test_dkss.py:185-193)
    t = ref["toy_plans"][0]
    assert (t["M"], t["m"]) == (2, 2)


@pytest.mark.parametrize("bits", [1024, 3000, 1 << 14, 1 << 16, 100_000])
def test_oracle_dmul_random(bits):
    rng = random.Random(bits)
    pl = P.dkss_select_params(bits)
    o = OraclePlan(pl)
    for _ in range(2):
        a = rng.getrandbits(bits) | 1 << (bits - 1)
        b = rng.getrandbits(bits)
        assert o.dmul(a, b) == a * b
