import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def iter_packed(d):
    """Unpack a make_golden.py instance pack into per-instance dicts."""
    G, E = d["G"], d["E"]
    om = oh = os_ = 0
    for i in range(len(G)):
        g, e = int(G[i]), int(E[i])
        m = d["m"][om : om + g * e].reshape(g, e)
        home = d["home"][oh : oh + e]
        S = d["S"][os_ : os_ + g * e * g].reshape(g, e, g)
        om += g * e
        oh += e
        os_ += g * e * g
        yield dict(m=m, home=home, q=int(d["q"][i]), S=S, iters=int(d["iters"][i]), i=i)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))

    return load
