import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test (oracle convergence legs)")


@pytest.fixture(scope="session")
def ora():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.hookimpl(trylast=True)
def pytest_collection_modifyitems(session, config, items):
    """Start the full-horizon oracle jobs (tests/_horizon.py) in the background when their tests
    are selected (after -m deselection) and a GPU is present, so they overlap the GPU suite."""
    if not any("test_zz_full_horizon_gpu" in it.nodeid for it in items):
        return
    try:
        import torch
        if not torch.cuda.is_available():
            return
    except Exception:
        return
    from tests import _horizon
    _horizon.start()
