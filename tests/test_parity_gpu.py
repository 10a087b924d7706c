"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded
inputs (BASELINE.json tolerances: fp64 normwise <= 1e-12 after 1 step, <= 1e-8 after 1000 steps on
configs[0]; diagnostics within 1e-12 relative; fp32 configs[4] <= 1e-4 after 100 steps)."""
import numpy as np
import pytest

from paper_2312_05410_b200 import pf
from tests import inputs
from tests._maps import oracle_member, normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pf.lib()


def _sim(p, mode="single"):
    return pf.Simulation(p, mode)


def test_cfg1_initial_fields_bitwise(ora):
    p = pf.pf_default_params(1)
    m, ic = oracle_member(ora, p, 0)
    with _sim(p) as s:
        got = s.fields(0)
    want = ora.initial_fields(ic, 64, 64, 0)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_cfg1_one_step_and_1000_steps(ora):
    """configs[0]: <= 1e-12 after 1 step, <= 1e-8 after 1000 steps (north_star Tolerances)."""
    p = pf.pf_default_params(1)
    m, ic = oracle_member(ora, p, 0)
    u0 = ora.initial_fields(ic, 64, 64, 0)
    with _sim(p) as s:
        s.step(1)
        e1 = normwise(s.fields(0), ora.step(m, *u0, 1))
        assert e1 <= 1e-12, e1
        s.step(999)
        ref = ora.step(m, *u0, 1000)
        got = s.fields(0)
        e = normwise(got, ref)
        assert e <= 1e-8, e
        d = s.diagnostics(0)
        dref = ora.diagnostics(m, *ref)
        for k in range(4):
            assert abs(d[k] - dref[k]) <= 1e-12 * abs(dref[k]), (k, d[k], dref[k])
        assert d[4] == 0
        steps, t, y0, ny = s.info()
        assert steps == 1000 and abs(t - 1.0) < 1e-12 and y0 == 0 and ny == 64


@pytest.mark.parametrize("nx,ny,members", [(72, 40, 3), (100, 37, 2), (8, 8, 1), (33, 65, 2), (130, 18, 1)])
def test_ragged_grids_random_inputs(ora, nx, ny, members):
    """Ragged tails in x and y (not multiples of the 32 x 16 tile), minimum grid 8 x 8, several
    members with different rates, oblique deposition and unequal mobilities; inputs set through
    pf_set_fields from the shared seeded generator."""
    p = pf.pf_default_params(1).replace(nx=nx, ny=ny, n_members=members, theta_deg=63.0,
                                       M_A_bulk=1.5, M_B_bulk=0.5, M_A_surf=2.0, M_B_surf=0.8,
                                       rate_lo=0.5, rate_hi=2.0, rho_in=0.9, graph_steps=0, seed=11)
    with _sim(p) as s:
        u = [inputs.random_state(nx, ny, 100 + k, phi_kind="smooth") for k in range(members)]
        for k in range(members):
            s.set_fields(k, *u[k])
        s.step(1)
        for k in range(members):
            m, _ = oracle_member(ora, p, k)
            e = normwise(s.fields(k), ora.step(m, *u[k], 1))
            assert e <= 1e-12, (k, e)
        s.step(49)
        for k in range(members):
            m, _ = oracle_member(ora, p, k)
            ref = ora.step(m, *u[k], 50)
            e = normwise(s.fields(k), ref)
            assert e <= 1e-10, (k, e)
            d = s.diagnostics(k)
            dref = ora.diagnostics(m, *ref)
            for q in range(4):
                assert abs(d[q] - dref[q]) <= 1e-12 * abs(dref[q]) + 1e-300, (k, q, d[q], dref[q])


def test_cfg2_1000_steps(ora):
    p = pf.pf_default_params(2)
    m, ic = oracle_member(ora, p, 0)
    u0 = ora.initial_fields(ic, 256, 256, 0)
    with _sim(p) as s:
        s.step(1000)
        e = normwise(s.fields(0), ora.step(m, *u0, 1000))
    assert e <= 1e-8, e


def test_uniform_state_fixed_point_bitwise():
    p = pf.pf_default_params(1).replace(ic=pf.PF_IC_NONE, nx=40, ny=24, theta_deg=70.0)
    with _sim(p) as s:
        c = np.full((24, 40), 0.37); phi = np.full((24, 40), 0.81); rho = np.full((24, 40), p.rho_in)
        s.set_fields(0, c, phi, rho)
        s.step(7)
        g = s.fields(0)
    assert np.array_equal(g[0], c) and np.array_equal(g[1], phi) and np.array_equal(g[2], rho)


def test_dataset_sweeps_parity(ora):
    """Per-member deposition rate, angle (R-15, R-21) and species mobilities (R-23) -- the paper's
    dataset sweep -- on an ensemble: every member against the oracle with its own
    parameters after 1 step (<= 1e-12) and 60 steps (<= 1e-10)."""
    p = pf.pf_default_params(2).replace(nx=96, ny=64, ic_height=20.0, n_members=4, member_offset=10,
                                       theta_deg=50.0, theta_span=40.0, rate_lo=0.6, rate_hi=2.0,
                                       mob_lo=0.4, mob_hi=1.0, M_A_bulk=10.0, M_B_bulk=4.0, M_A_surf=8.0,
                                       M_B_surf=2.0, seed=31)
    with _sim(p) as s:
        s.step(1)
        g1 = [s.fields(k) for k in range(4)]
        s.step(59)
        g60 = [s.fields(k) for k in range(4)]
    for k in range(4):
        m, ic = oracle_member(ora, p, 10 + k)
        u0 = ora.initial_fields(ic, p.nx, p.ny, 10 + k)
        assert normwise(g1[k], ora.step(m, *u0, 1)) <= 1e-12, k
        assert normwise(g60[k], ora.step(m, *u0, 60)) <= 1e-10, k


def test_stochastic_inflow_parity(ora):
    """R-27 stochastic inflow (the kernels draw the truncated-Gaussian reservoir row of every step
    on the device): each member against the oracle's own generator and step after 1 step
    (<= 1e-12) and 40 steps (<= 1e-10); c mass unchanged (the inflow only feeds rho)."""
    p = pf.pf_default_params(2).replace(nx=64, ny=48, ic_height=16.0, n_members=3, member_offset=4,
                                       noise_rho=0.3, rho_in=1.0, theta_deg=70.0, seed=12, graph_steps=8)
    with _sim(p) as s:
        s.step(1)
        g1 = [s.fields(k) for k in range(3)]
        s.step(39)
        g40 = [s.fields(k) for k in range(3)]
        d = [s.diagnostics(k) for k in range(3)]
    for k in range(3):
        m, ic = oracle_member(ora, p, 4 + k)
        u0 = ora.initial_fields(ic, p.nx, p.ny, 4 + k)
        r1 = ora.step_inflow(m, *u0, 1, 0, 12, 4 + k, 0.3)
        r40 = ora.step_inflow(m, *u0, 40, 0, 12, 4 + k, 0.3)
        assert normwise(g1[k], r1) <= 1e-12, k
        assert normwise(g40[k], r40) <= 1e-10, k
        assert abs(d[k][0] - ora.diagnostics(m, *u0)[0]) <= 1e-12 * abs(d[k][0])
        # the noise is really there: the deterministic run differs
        assert normwise(g40[k], ora.step(m, *u0, 40)) > 1e-8


def test_regular_solution_parity(ora):
    """R-28 regular-solution composition energy on the device (fp64 log): each member against the
    oracle after 1 step (<= 1e-12) and 80 steps (<= 1e-10); mass and energy diagnostics (the energy
    uses the same free energy) within 1e-12."""
    p = pf.pf_default_params(2).replace(nx=80, ny=48, ic_height=16.0, n_members=2, fe_model=1, omega=2.5,
                                       temp_rs=0.5, theta_deg=75.0, M_A_bulk=6.0, M_B_bulk=3.0, seed=19, dt=4e-4)
    with _sim(p) as s:
        s.step(1)
        g1 = [s.fields(k) for k in range(2)]
        s.step(79)
        g80 = [s.fields(k) for k in range(2)]
        d = [s.diagnostics(k) for k in range(2)]
    for k in range(2):
        m, ic = oracle_member(ora, p, k)
        u0 = ora.initial_fields(ic, p.nx, p.ny, k)
        assert normwise(g1[k], ora.step(m, *u0, 1)) <= 1e-12, k
        r80 = ora.step(m, *u0, 80)
        assert normwise(g80[k], r80) <= 1e-10, k
        dref = ora.diagnostics(m, *r80)
        for q in (0, 3):
            assert abs(d[k][q] - dref[q]) <= 1e-12 * abs(dref[q]), (k, q, d[k][q], dref[q])
