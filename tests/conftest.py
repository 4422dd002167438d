"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` runs on a B200."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port

    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref/libattnkit_ref.so not built (make -C oracle ref)")
    return Reference()


@pytest.fixture(scope="session")
def dfa():
    import paper_2403_09195_b200 as dfa_mod

    return dfa_mod


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda:0")


def rand(shape, seed, dtype=np.float64):
    """Inputs for parity runs: numpy PCG64, reproducible on any host."""
    return np.random.default_rng(seed).standard_normal(shape).astype(dtype)
