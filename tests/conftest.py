import os
import random
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdkss.so")


@pytest.fixture(autouse=True)
def _default_word_size():
    # every test starts from the 64-bit build unless it switches explicitly (mirrors the
    # reference's tests/conftest.py:8-13)
    from paper_1503_04955_b200.words import set_word_bits

    set_word_bits(64)
    yield
    set_word_bits(64)


@pytest.fixture
def rng():
    return random.Random(0xC0FFEE)


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def cuda_ok():
    try:
        import torch

        ok = torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        ok = False
    if not ok:
        pytest.skip("no CUDA device")
    return True
