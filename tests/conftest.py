import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libbfly.so")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def chain_from_golden(d, prefix=""):
    from oracle.chain import Chain
    p = prefix
    g_lvls = [int(x) for x in d[p + "g_lvls"]]
    h_lvls = [int(x) for x in d[p + "h_lvls"]]
    return Chain(int(d[p + "n"]), int(d[p + "levels"]), int(d[p + "rank"]), d[p + "u_leaf"],
                 [(l, d[f"{p}g_{l}"]) for l in g_lvls], d[p + "weights"],
                 [(l, d[f"{p}h_{l}"]) for l in h_lvls], d[p + "v_leaf"])


def complex_gaussian(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.fixture
def rng():
    return np.random.default_rng(20240801)
