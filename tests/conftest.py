import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref/liblqref.so not built (reference sources absent)")
    return oracle.Ref()


@pytest.fixture(scope="session")
def lqg():
    import paper_2509_01229_b200 as lqg
    lqg._lib.lib()
    return lqg


def make_weights(rng, n, k, std=0.02, outliers=True):
    w = (rng.standard_normal((n, k)) * std).astype(np.float32)
    if outliers and n * k >= 64:
        idx = rng.choice(n * k, size=max(1, n * k // 1000), replace=False)
        w.reshape(-1)[idx] *= 20
    return w


def make_acts(rng, m, k, outliers=True):
    x = rng.standard_normal((m, k)).astype(np.float32)
    if outliers:
        idx = rng.choice(m * k, size=max(1, m * k // 1000), replace=False)
        x.reshape(-1)[idx] *= 20
    return x
