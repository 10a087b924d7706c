"""NEXT-1: the trajectory / dataset driver pf_trajectory -- composite snapshots of
an ensemble with per-member deposition rates and angles (v in [0.3, 1], theta in
[50, 90] degrees; 50 equally spaced snapshots).

* GPU-vs-GPU: every snapshot is bitwise the composite of the fields pf_get_fields returns after
  the same number of steps, the snapshot times form the arithmetic sequence t0 + s dt steps_between
  (SPEC S:249-251), and slab decompositions give the same trajectory.
* GPU-vs-oracle: composites of the oracle's fields after the same steps, each member with its own
  velocity (R-15, R-21), within 1e-12 normwise; cells whose phi lies within 1e-9 of 1/2 are
  excluded from the comparison (the solid / vapour decision is not unique there).
"""
import numpy as np
import pytest

from paper_2312_05410_b200 import pf
from tests._maps import oracle_member, normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pf.lib()


def _params(**kw):
    p = pf.pf_default_params(2).replace(nx=96, ny=64, ic_height=20.0, n_members=5, theta_deg=50.0,
                                       theta_span=40.0, rate_lo=0.6, rate_hi=2.0, seed=77, check_every=7)
    return p.replace(**kw)


def _composite(c, phi):
    return np.where(phi > 0.5, c, 0.0)


@pytest.mark.parametrize("mode", ["single", ("loopback", 4)])
def test_trajectory_equals_step_by_step(mode):
    p = _params()
    S, K = 6, 9
    with pf.Simulation(p, mode) as s:
        out = np.full((p.n_members, S, p.ny, p.nx), np.nan)
        times = np.zeros(S)
        s.step(3)
        pf.pf_trajectory(s.ctx, S, K, out, times)
        assert s.info()[0] == 3 + (S - 1) * K
    with pf.Simulation(p) as s:
        s.step(3)
        for k in range(S):
            if k:
                s.step(K)
            c, phi, _ = s.fields(-1)
            assert np.array_equal(out[:, k], _composite(c, phi)), k
    dt = p.dt
    assert np.allclose(times, (3 + K * np.arange(S)) * dt, rtol=0, atol=1e-15)
    assert np.all(np.diff(times) > 0)


def test_trajectory_against_oracle(ora):
    p = _params()
    S, K = 5, 20
    with pf.Simulation(p) as s:
        out = np.empty((p.n_members, S, p.ny, p.nx))
        pf.pf_trajectory(s.ctx, S, K, out)
    for k in range(p.n_members):
        m, ic = oracle_member(ora, p, k)
        u = ora.initial_fields(ic, p.nx, p.ny, k)
        for q in range(S):
            if q:
                u = ora.step(m, *u, K)
            ref = ora.composite(u[0], u[1])
            keep = np.abs(u[1] - 0.5) > 1e-9
            got = np.where(keep, out[k, q], 0.0)
            want = np.where(keep, ref, 0.0)
            assert normwise([got], [want]) <= 1e-12, (k, q)
            # the angle sweep really varies the deposition direction between members
    vel = [pf.pf_member_velocity(p, k) for k in range(p.n_members)]
    assert len({round(np.degrees(np.arctan2(-vy, vx)), 6) for vx, vy in vel}) == p.n_members


def test_trajectory_single_snapshot_takes_no_steps():
    p = _params(n_members=2)
    with pf.Simulation(p) as s:
        out = np.empty((2, 1, p.ny, p.nx))
        pf.pf_trajectory(s.ctx, 1, 100, out)
        assert s.info()[0] == 0
        c, phi, _ = s.fields(-1)
        assert np.array_equal(out[:, 0], _composite(c, phi))


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_trajectory_file_equals_trajectory(tmp_path, dtype):
    """pf_trajectory_file (the streamed trajectory file of NEXT-1) holds exactly pf_trajectory's
    snapshots (float32: the rounded values), the member records, the snapshot times, and leaves the
    ctx at the same step."""
    p = _params()
    S, K = 7, 5
    with pf.Simulation(p) as s:
        s.step(2)
        ref = np.empty((p.n_members, S, p.ny, p.nx))
        tref = np.zeros(S)
        pf.pf_trajectory(s.ctx, S, K, ref, tref)
    path = str(tmp_path / f"traj_{dtype}.pftraj")
    with pf.Simulation(p) as s:
        s.step(2)
        pf.pf_trajectory_file(s.ctx, path, S, K, dtype)
        assert s.info()[0] == 2 + (S - 1) * K
    h, recs, snaps, times = pf.read_trajectory(path)
    assert (h["members"], h["n_snapshots"], h["ny_rows"], h["nx"], h["step0"], h["steps_between"]) == \
        (p.n_members, S, p.ny, p.nx, 2, K)
    want = ref.transpose(1, 0, 2, 3)
    if dtype == "float64":
        assert np.array_equal(np.asarray(snaps), want)
    else:
        assert np.array_equal(np.asarray(snaps), want.astype(np.float32))
    assert np.array_equal(times, tref)
    for m in range(p.n_members):
        assert recs[m, 0] == m
        assert (recs[m, 1], recs[m, 2]) == pf.pf_member_velocity(p, m)
