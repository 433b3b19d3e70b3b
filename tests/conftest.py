import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (run on the B200 box)")


@pytest.fixture(scope="session")
def oracle():
    """CPU parity oracle: .port = C restatement, .ref = compiled unmodified reference (or None)."""
    import oracle as orc
    return orc


@pytest.fixture(scope="session")
def port(oracle):
    return oracle.port


@pytest.fixture(scope="session")
def ref(oracle):
    r = oracle.ref
    if r is None:
        pytest.skip("oracle/_ref/libskinnyqr_ref.so not built")
    return r


@pytest.fixture(scope="session")
def sq():
    import paper_2603_20889_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def ctx(sq):
    return sq.default_context(0)


def gaussian(m, n, seed=0):
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((m, n)))


def normalize(r):
    r = np.array(r, dtype=np.float64, order="F")
    for i in range(r.shape[0]):
        if r[i, i] < 0.0:
            r[i, i:] = -r[i, i:]
    return r


EPS = np.finfo(np.float64).eps


def r_bound(x, c=64.0):
    """north_star: R agrees up to signs within c*n*eps*|X|_F (c = 64)."""
    return c * x.shape[1] * EPS * np.linalg.norm(x)
