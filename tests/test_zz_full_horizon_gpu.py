"""Full-horizon GPU parity (BASELINE north_star "Tolerances"): the whole
configs[1] run (256^2, the paper's mesh P:353, 10,000 steps) and configs[2] members 0, 21, 42, 63
over the full 5,000 steps, every cell, normwise <= 1e-8 (R-17), with the mass of c conserved.
The oracle runs were started in the background at collection (tests/_horizon.py); this file is
named to run last so that they overlap the rest of the suite."""
import numpy as np
import pytest

from paper_2312_05410_b200 import pf
from tests import _horizon
from tests._maps import normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pf.lib()


def test_cfg2_full_horizon_10000_steps():
    p = pf.pf_default_params(2)
    with pf.Simulation(p) as s:
        d0 = s.diagnostics(0)
        s.step(_horizon.CFG2_STEPS)
        got = s.fields(0)
        d1 = s.diagnostics(0)
        assert s.info()[0] == _horizon.CFG2_STEPS
    ref = _horizon.result("cfg2")
    e = normwise(got, ref)
    print(f"configs[1] after {_horizon.CFG2_STEPS} steps: normwise {e:.3e}")
    assert e <= 1e-8, e
    assert abs(d1[0] - d0[0]) <= 1e-12 * abs(d0[0])
    assert d1[4] == 0


def test_cfg3_members_full_horizon_5000_steps():
    p = pf.pf_default_params(3)
    with pf.Simulation(p) as s:
        s.step(_horizon.CFG3_STEPS)
        got = {k: s.fields(k) for k in _horizon.CFG3_MEMBERS}
    for k in _horizon.CFG3_MEMBERS:
        e = normwise(got[k], _horizon.result(("cfg3", k)))
        print(f"configs[2] member {k} after {_horizon.CFG3_STEPS} steps: normwise {e:.3e}")
        assert e <= 1e-8, (k, e)
        assert np.all(np.isfinite(got[k][0]))
