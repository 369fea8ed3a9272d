"""Shared fixtures. Tests marked `gpu` need a CUDA device (run on a B200 with
`pytest -m gpu`); everything else runs on CPU (`pytest -m "not gpu"`)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz")))


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    try:
        return oracle.Reference()
    except (FileNotFoundError, OSError) as e:  # pragma: no cover
        pytest.skip(f"reference library unavailable: {e}")


@pytest.fixture(scope="session")
def tq():
    import paper_2205_02646_b200 as tq
    return tq


@pytest.fixture(scope="session")
def need_gpu(tq):
    if tq.device_count() < 1:
        pytest.fail("gpu-marked test ran without a CUDA device")
    return True
