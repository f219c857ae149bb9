"""mul()/ALGORITHMS routing mirrors bigmul/dispatch.py:11-46 (no GPU needed)."""
import pytest

from paper_1503_04955_b200 import ALGORITHMS, Natural, ThresholdTable, dmul, mul


def test_algorithm_table_names():
    assert set(ALGORITHMS) == {"omul", "kmul", "t3mul", "qmul", "smul", "dmul"}


def test_unknown_algorithm():
    with pytest.raises(ValueError):
        mul(3, 5, algorithm="fft")


def test_out_of_scope_rungs_raise():
    with pytest.raises(NotImplementedError):
        mul(3, 5, algorithm="t3mul")
    with pytest.raises(NotImplementedError):
        mul(3, 5)  # default ladder would pick omul


def test_thresholds_validated():
    with pytest.raises(ValueError):
        mul(3, 5, thresholds=ThresholdTable(kmul=200, t3mul=100), algorithm="dmul")


def test_dmul_zero_shortcut_needs_no_device():
    a = Natural.from_int(0xDEAD, length=2)
    r = dmul(a, 0)
    assert r.to_int() == 0 and len(r) == 3     # bigmul/dkss.py:529-531
    r = mul(0, a, algorithm="dmul")
    assert r.to_int() == 0


def test_smul_zero_shortcut_needs_no_device():
    r = mul(Natural.from_int(7, length=3), 0, algorithm="smul")  # bigmul/smul.py:290-292
    assert r.to_int() == 0 and len(r) == 4


def test_dmul_argument_types():
    with pytest.raises(TypeError):
        dmul(1.0, 2)
    with pytest.raises(ValueError):
        dmul(-5, 2)
