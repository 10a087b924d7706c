"""NEXT-2 on the GPU (pf_s2 / pf_s2_rel_l2: cuFFT + own kernels) against the oracle's statistics
(oracle.s2_fft / radial_average / rel_l2, themselves pinned to the brute-force double sum and closed
forms in tests/test_oracle_stats.py), on composite snapshots of a real trajectory."""
import numpy as np
import pytest

from paper_2312_05410_b200 import pf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pf.lib()


def test_s2_closed_forms_gpu(ora):
    ones = np.ones((2, 16, 24))
    s2, rad = pf.pf_s2(ones)
    assert np.abs(s2 - 1.0).max() < 1e-14 and np.abs(rad - 1.0).max() < 1e-14
    one = np.zeros((16, 16)); one[5, 9] = 0.7
    s2, rad = pf.pf_s2(one)
    assert abs(s2[8, 8] - 1.0 / 256) < 1e-17 and np.abs(np.delete(s2.ravel(), 8 * 16 + 8)).max() < 1e-17


def test_s2_of_trajectory_matches_oracle(ora):
    p = pf.pf_default_params(2).replace(nx=96, ny=64, ic_height=24.0, n_members=2, rate_lo=0.6, rate_hi=2.0,
                                       theta_deg=50.0, theta_span=40.0, seed=5)
    with pf.Simulation(p) as s:
        out = np.empty((2, 4, 64, 96))
        pf.pf_trajectory(s.ctx, 4, 40, out)
    comp = out.reshape(8, 64, 96)
    s2, rad = pf.pf_s2(comp)
    for b in range(8):
        want = ora.s2_fft(ora.indicator(comp[b]))
        assert np.abs(s2[b] - want).max() < 1e-12, b
        assert np.abs(rad[b] - ora.radial_average(want)).max() < 1e-12, b
        assert s2[b][32, 48] == pytest.approx(ora.indicator(comp[b]).mean(), abs=1e-14)
    r = pf.pf_s2_rel_l2(comp[:4], comp[4:])
    for b in range(4):
        want = ora.rel_l2(ora.s2_fft(ora.indicator(comp[b])), ora.s2_fft(ora.indicator(comp[4 + b])))
        assert r[b] == pytest.approx(want, rel=1e-10, abs=1e-14)
    assert np.all(pf.pf_s2_rel_l2(comp, comp) == 0.0)
