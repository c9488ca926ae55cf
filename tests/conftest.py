import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running full-size parity check")


from __graft_entry__ import ensure_built  # noqa: E402

ensure_built()


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN, allow_pickle=False))


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def sb():
    import paper_2410_14056_b200 as sb
    return sb


def golden_graph(golden, name):
    import paper_2410_14056_b200 as sb
    return sb.Graph(golden[f"g/{name}/off"], golden[f"g/{name}/adj"])


@pytest.fixture(scope="session")
def gpu_available():
    import paper_2410_14056_b200._lib as L
    return L.lib().saba_cu_device_count() > 0


def pytest_collection_modifyitems(config, items):
    import paper_2410_14056_b200._lib as L
    if L.lib().saba_cu_device_count() > 0:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this environment")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
