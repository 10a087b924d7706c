"""Pins of the oracle's seeded input generator (readings R-14, R-15, R-16)."""
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_published_values(ora):
    with open(os.path.join(GOLDEN, "splitmix64.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            z, want = (int(t, 16) for t in line.split())
            assert ora.sm64(z) == want


def test_uniform_and_gauss_statistics(ora):
    u = np.array([ora.uniform(9, 4, k) for k in range(20000)])
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.01 and abs(u.var() - 1 / 12) < 0.003
    z = np.array([ora.gauss(9, 5, k) for k in range(20000)])
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1) < 0.03
    # streams differ, draws are reproducible
    assert ora.uniform(9, 4, 3) == ora.uniform(9, 4, 3)
    assert ora.uniform(9, 4, 3) != ora.uniform(9, 5, 3)


def test_film_recipe(ora):
    """cfg1 (BASELINE configs[0]): phi = [y<16] + U(+-0.01); c = 0.5 + U(+-0.05); rho = rho_in above."""
    pr = ora.preset(1)
    c, phi, rho = ora.initial_fields(pr["ic"], 64, 64, 0)
    solid = (np.arange(64)[:, None] < 16) * np.ones((1, 64))
    assert np.max(np.abs(phi - solid)) <= 0.01
    assert np.max(np.abs(c - 0.5)) <= 0.05
    assert np.array_equal(rho, 1.0 - solid)
    assert abs((c - 0.5).mean()) < 2e-3


def test_rough_recipe(ora):
    """cfg2 (configs[1]): substrate height 32, roughness amplitude 2, wavelength 32; c ~ N(0.5, 0.05^2)."""
    pr = ora.preset(2)
    c, phi, rho = ora.initial_fields(pr["ic"], 256, 256, 0)
    i = np.arange(256)[None, :]; j = np.arange(256)[:, None]
    H = 32 + 2 * np.sin(2 * np.pi * i / 32)
    want = 0.5 * (1 - np.tanh((j - H) / math.sqrt(2.0)))
    np.testing.assert_allclose(phi, want, atol=1e-15)
    np.testing.assert_allclose(rho, 1 - phi, atol=1e-15)
    assert abs(c.mean() - 0.5) < 1e-3 and abs(c.std() - 0.05) < 1e-3


def test_columns_recipe(ora):
    """cfg5 (configs[4]): 64 columns of random width, c alternating 0.2 / 0.8, tanh film at ny/2."""
    ic = ora.preset(5)["ic"]
    nx, ny = 1024, 16
    ic.height = ny / 2
    c, phi, rho = ora.initial_fields(ic, nx, ny, 0)
    row = c[0]
    assert np.all(c == row[None, :])
    runs = 1 + np.count_nonzero(np.diff(row))
    assert runs == 64
    assert row[0] == 0.2 and set(np.unique(row)) == {0.2, 0.8}
    starts = np.flatnonzero(np.diff(row)) + 1
    assert np.all(np.diff(row[np.r_[0, starts]]) != 0)


def test_member_rates(ora):
    """cfg3 (configs[2]): per-member rates uniform in [0.5, 2] x nominal v0 = 0.5; theta = 90 deg."""
    ic = ora.preset(3)["ic"]
    v = np.array([ora.member_velocity(ic, m) for m in range(64)])
    assert np.all(np.abs(v[:, 0]) < 1e-15)
    sp = -v[:, 1]
    assert sp.min() >= 0.25 and sp.max() <= 1.0 and sp.std() > 0.1
    assert len(set(sp)) == 64
    ic1 = ora.preset(1)["ic"]
    assert ora.member_velocity(ic1, 0)[1] == -0.5


def test_member_angle_sweep_pins(ora):
    """R-21: theta_m = theta_deg + theta_span U(seed, 8m+4, 0).  The velocity direction recovered
    with atan2 lies in [50, 90) degrees for the paper's sweep, its mean over many members is
    the interval's midpoint, the speed is the member's rate (R-15), and theta_span = 0 reproduces the
    fixed-angle velocity bit for bit."""
    import math
    ic = ora.IC(kind="rough", v0=0.5, theta_deg=50.0, theta_span=40.0, rate_lo=0.6, rate_hi=2.0, seed=9)
    angs = []
    for m in range(2000):
        vx, vy = ora.member_velocity(ic, m)
        a = math.degrees(math.atan2(-vy, vx))
        assert 50.0 - 1e-9 <= a < 90.0 + 1e-9
        u = ora.uniform(9, 8 * m + 3, 0)
        assert math.isclose(math.hypot(vx, vy), 0.5 * (0.6 + 1.4 * u), rel_tol=1e-14)
        angs.append(a)
    assert abs(sum(angs) / len(angs) - 70.0) < 1.0
    fixed = ora.IC(kind="rough", v0=0.5, theta_deg=63.0, theta_span=0.0, seed=9)
    vx, vy = ora.member_velocity(fixed, 5)
    u = ora.uniform(9, 8 * 5 + 3, 0)
    th = 63.0 * (math.pi / 180.0)
    assert vx == 0.5 * (1.0 + 0.0 * u) * math.cos(th) and vy == -(0.5 * (1.0 + 0.0 * u) * math.sin(th))


def test_composite_definition(ora):
    """Composite snapshot field: c in the solid (phi > 1/2), exactly 0 in the vapour; phi = 1/2 is
    vapour (strict inequality)."""
    import numpy as np
    c = np.array([[0.3, 0.7, 0.5], [0.2, 0.9, 0.4]])
    phi = np.array([[1.0, 0.5000000001, 0.5], [0.0, 0.49, 2.0]])
    want = np.array([[0.3, 0.7, 0.0], [0.0, 0.0, 0.4]])
    assert np.array_equal(ora.composite(c, phi), want)


def test_member_mobility_sweep_pins(ora):
    """R-23: species-mobility multipliers a (stream 8m+5) and b (stream 8m+6) are the affine maps
    of the counter generator's uniforms onto [mob_lo, mob_hi); no sweep gives exactly 1."""
    ic = ora.IC(kind="rough", mob_lo=0.5, mob_hi=2.0, seed=4)
    A, B = [], []
    for m in range(3000):
        a, b = ora.member_mobility(ic, m)
        assert a == 0.5 + 1.5 * ora.uniform(4, 8 * m + 5, 0)
        assert b == 0.5 + 1.5 * ora.uniform(4, 8 * m + 6, 0)
        assert 0.5 <= a < 2.0 and 0.5 <= b < 2.0
        A.append(a); B.append(b)
    import numpy as np
    assert abs(np.mean(A) - 1.25) < 0.03 and abs(np.mean(B) - 1.25) < 0.03
    assert abs(np.corrcoef(A, B)[0, 1]) < 0.06
    assert ora.member_mobility(ora.IC(kind="rough", seed=4), 7) == (1.0, 1.0)


def test_stochastic_inflow_pins(ora):
    """R-27: per-step, per-column truncated Gaussian N(rho_in, sigma^2) on [0, 2 rho_in].
    sigma = 0 gives rho_in exactly; small sigma gives mean rho_in and standard deviation sigma (the
    truncation is inactive); large sigma keeps every value inside the bounds; draws differ between
    steps, columns and members; a zero-noise run equals the deterministic run bit for bit."""
    import numpy as np
    assert ora.inflow(3, 2, 10, 64, 5, 0.8, 0.0) == 0.8
    v = np.array([ora.inflow(3, 2, s, 64, i, 1.0, 0.05) for s in range(100) for i in range(64)])
    assert abs(v.mean() - 1.0) < 3 * 0.05 / np.sqrt(v.size) * 2 and abs(v.std() - 0.05) < 0.003
    w = np.array([ora.inflow(3, 2, s, 64, i, 1.0, 2.0) for s in range(50) for i in range(64)])
    assert w.min() >= 0.0 and w.max() <= 2.0 and abs(w.mean() - 1.0) < 0.05
    assert ora.inflow(3, 2, 7, 64, 5, 1.0, 0.1) != ora.inflow(3, 2, 8, 64, 5, 1.0, 0.1)
    assert ora.inflow(3, 2, 7, 64, 5, 1.0, 0.1) != ora.inflow(3, 3, 7, 64, 5, 1.0, 0.1)
    m = ora.Model(nx=16, ny=12, v_y=-0.5)
    g = np.random.default_rng(0)
    u = (0.5 + 0.05 * g.random((12, 16)), g.random((12, 16)), g.random((12, 16)))
    a = ora.step(m, *u, 5)
    b = ora.step_inflow(m, *u, 5, 0, 3, 2, 0.0)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
