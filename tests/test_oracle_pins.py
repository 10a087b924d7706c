"""Pins of the CPU oracle against things other than itself.

Every test here runs on the CPU (no GPU marker).  The expected values come from
the paper / SPEC worked examples (tests/golden/), closed forms of the discrete
operators, invariants of the scheme, or brute-force linear algebra written in
this file.  None of them comes from the CUDA path.
"""
import math
import os
from dataclasses import replace

import numpy as np
import pytest

from tests import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _model(ora, **kw):
    return replace(ora.Model(), **kw)


# --------------------------------------------------------------------------- golden values
def _golden_rows():
    rows = []
    with open(os.path.join(GOLDEN, "constitutive_points.txt")) as f:
        for line in f:
            line = line.split("|")[0].strip()
            if not line or line.startswith("#"):
                continue
            tok = line.split()
            rows.append((tok[0], [float(t) for t in tok[1:-1]], float(tok[-1])))
    return rows


@pytest.mark.parametrize("row", _golden_rows(), ids=lambda r: f"{r[0]}{r[1]}")
def test_constitutive_golden(ora, row):
    """S:168-185 worked examples of switching_h / mobility_c (mapped through R-1)."""
    fn, args, want = row
    if fn == "h":
        got = ora.h(args[0])
    elif fn == "p":
        got = ora.p(args[0])
    elif fn == "e":
        got = ora.e(args[0], args[1])
    elif fn == "mob":
        m = _model(ora, MA_bulk=3.0, MB_bulk=5.0, MA_surf=7.0, MB_surf=11.0, sigma_surf=1.0)
        got = ora.mobility_c(m, args[0], args[1])
    assert got == pytest.approx(want, rel=1e-15, abs=1e-300)


def test_p_equals_smoothstep_in_phi(ora):
    """R-1: 1/4 (2 - phit)(1 + phit)^2 == phi^2 (3 - 2 phi) for phit = 2 phi - 1."""
    for phi in np.linspace(-0.2, 1.2, 57):
        assert ora.p(phi) == pytest.approx(phi * phi * (3 - 2 * phi), abs=4e-16)


def test_h_properties(ora):
    """S:172 post: h(0)=0, h(1)=1, h'(0)=h'(1)=0, monotone on [0,1]."""
    xs = np.linspace(0, 1, 1001)
    hs = np.array([ora.h(x) for x in xs])
    assert np.all(np.diff(hs) >= 0)
    eps = 1e-6
    assert abs(ora.h(eps) - ora.h(0)) / eps < 1e-5
    assert abs(ora.h(1) - ora.h(1 - eps)) / eps < 1e-5


# --------------------------------------------------------------------------- operators
def test_laplacian_symbols(ora):
    """Stencil symbols: periodic cos(2 pi m i/nx) and the Neumann (mirror) eigenvector
    cos(pi m (j+1/2)/ny); reservoir mode cos(k (j+1/2)), k = pi(q+1/2)/(ny+1/2)."""
    nx, ny, dx = 32, 24, 0.7
    i = np.arange(nx)[None, :]
    j = np.arange(ny)[:, None]
    for m in (1, 3, 7):
        u = np.cos(2 * np.pi * m * i / nx) * np.ones((ny, 1))
        lam = 4 / dx**2 * math.sin(math.pi * m / nx) ** 2
        np.testing.assert_allclose(ora.laplacian(u, dx), -lam * u, atol=1e-13)
        v = np.cos(np.pi * m * (j + 0.5) / ny) * np.ones((1, nx))
        lam = 4 / dx**2 * math.sin(math.pi * m / (2 * ny)) ** 2
        np.testing.assert_allclose(ora.laplacian(v, dx), -lam * v, atol=1e-13)
    for q in (0, 2, 5):
        k = np.pi * (q + 0.5) / (ny + 0.5)
        rho_in = 0.8
        w = rho_in + 0.3 * np.cos(k * (j + 0.5)) * np.ones((1, nx))
        lam = 4 / dx**2 * math.sin(k / 2) ** 2
        np.testing.assert_allclose(ora.laplacian(w, dx, ora.RESERVOIR, rho_in), -lam * (w - rho_in),
                                   atol=1e-13)


def test_laplacian_quadratic_and_gradient_linear(ora):
    """the 5-point stencil is exact on quadratics (interior); central G exact on linears."""
    nx, ny, dx = 16, 16, 1.0
    y = np.arange(ny)[:, None] * np.ones((1, nx))
    L = ora.laplacian(y**2, dx)
    np.testing.assert_allclose(L[1:-1], 2.0, atol=1e-12)
    gx, gy = ora.gradient(3.0 * y + 1.0, dx)
    np.testing.assert_allclose(gy[1:-1], 3.0, atol=1e-13)
    np.testing.assert_allclose(gx, 0.0, atol=1e-13)
    # mirror rule: at j=0 the ghost u[-1]=u[0]
    np.testing.assert_allclose(gy[0], (3.0 * 1 + 1 - 1.0) / 2, atol=1e-13)


def _face_matrix(nx, ny):
    """Face-difference matrix D (faces x cells): (D u)_f = u_b - u_a over every periodic
    x-face and the ny-1 interior y-face rows; no y-boundary faces (R-8, R-12)."""
    N = nx * ny
    rows, ia, ib = [], [], []
    for j in range(ny):
        for i in range(nx):
            ia.append(j * nx + i); ib.append(j * nx + (i + 1) % nx)
    for j in range(ny - 1):
        for i in range(nx):
            ia.append(j * nx + i); ib.append((j + 1) * nx + i)
    D = np.zeros((len(ia), N))
    for f, (a, b) in enumerate(zip(ia, ib)):
        D[f, a] -= 1.0
        D[f, b] += 1.0
    return D, np.array(ia), np.array(ib)


def test_rhs_dense_brute_force_8x8(ora):
    """8x8 brute force: L = -D^T D/dx^2, R_c = -D^T diag(M_f) D mu_c/dx^2 with
    M_f = (M_a + M_b)/2, R_phi = M_phi L mu_phi + S, R_rho = D_rho L_res rho - v.G rho
    - rho v.G phit with phit = 2 phi - 1 (P:340 in the paper's variable; R-1, R-9).
    Assembled as dense matrices, independent of the stencil loops."""
    nx = ny = 8
    dx = 0.9
    D, ia, ib = _face_matrix(nx, ny)
    Lmat = -(D.T @ D) / dx**2
    # central gradient matrices with mirror y rule
    N = nx * ny
    Gx = np.zeros((N, N)); Gy = np.zeros((N, N))
    for j in range(ny):
        for i in range(nx):
            k = j * nx + i
            Gx[k, j * nx + (i + 1) % nx] += 1 / (2 * dx)
            Gx[k, j * nx + (i - 1) % nx] -= 1 / (2 * dx)
            jp = j + 1 if j + 1 < ny else ny - 1
            jm = j - 1 if j - 1 >= 0 else 0
            Gy[k, jp * nx + i] += 1 / (2 * dx)
            Gy[k, jm * nx + i] -= 1 / (2 * dx)
    # reservoir-rule operators for rho: top ghost = rho_in (affine)
    rho_in = 0.7
    Lres = Lmat.copy(); bres = np.zeros(N)
    Gyres = Gy.copy(); gres = np.zeros(N)
    for i in range(nx):
        k = (ny - 1) * nx + i
        # mirror contributed 0 for the top face; reservoir adds (rho_in - rho_k)/dx^2
        Lres[k, k] -= 1 / dx**2
        bres[k] += rho_in / dx**2
        # Gy row at top: mirror used +u[ny-1]; reservoir uses rho_in instead
        Gyres[k, k] -= 1 / (2 * dx)
        gres[k] += rho_in / (2 * dx)
    for seed in range(3):
        g = np.random.default_rng(100 + seed)
        c = g.random((ny, nx)); phi = g.random((ny, nx)); rho = g.random((ny, nx))
        m = _model(ora, dx=dx, MA_bulk=1.3, MB_bulk=0.4, MA_surf=2.1, MB_surf=0.9, sigma_surf=0.6,
                   M_phi=1.7, D_rho=0.8, rho_in=rho_in, v_x=0.23, v_y=-0.41, kappa_c=0.9,
                   kappa_phi=1.1, W_c=1.2, W_phi=0.8)
        mu_c, mu_p = ora.mu(m, c, phi)
        M = ora.mobility_field(m, c, phi).ravel()
        Mf = 0.5 * (M[ia] + M[ib])
        Rc_bf = -(D.T @ (Mf * (D @ mu_c.ravel()))) / dx**2
        S_bf = rho.ravel() * (m.v_x * (Gx @ phi.ravel()) + m.v_y * (Gy @ phi.ravel()))
        phit = 2.0 * phi.ravel() - 1.0
        Rp_bf = m.M_phi * (Lmat @ mu_p.ravel()) + S_bf
        Rr_bf = (m.D_rho * (Lres @ rho.ravel() + bres)
                 - (m.v_x * (Gx @ rho.ravel()) + m.v_y * (Gyres @ rho.ravel() + gres))
                 - rho.ravel() * (m.v_x * (Gx @ phit) + m.v_y * (Gy @ phit)))
        Rc, Rp, Rr, S = ora.rhs(m, c, phi, rho)
        for got, want in ((Rc, Rc_bf), (Rp, Rp_bf), (Rr, Rr_bf), (S, S_bf)):
            assert np.max(np.abs(got.ravel() - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))
        # the Laplacian inside mu equals the matrix one
        lc = (Lmat @ c.ravel()).reshape(ny, nx)
        np.testing.assert_allclose(ora.laplacian(c, dx), lc, atol=1e-13)


# --------------------------------------------------------------------------- variational identity
def _energy_complex(m, c, phi):
    """E_h written from F (R-2): dx^2 sum f + sum_interior_faces kappa/2 (du)^2, complex-safe."""
    f = m.W_c * c**2 * (1 - c) ** 2 * phi + m.W_phi * phi**2 * (1 - phi) ** 2
    E = m.dx**2 * f.sum()
    for u, k in ((c, m.kappa_c), (phi, m.kappa_phi)):
        dxu = np.roll(u, -1, axis=1) - u
        dyu = u[1:, :] - u[:-1, :]
        E = E + 0.5 * k * ((dxu**2).sum() + (dyu**2).sum())
    return E


def test_mu_is_variational_derivative_complex_step(ora):
    """mu = (1/dx^2) dE_h/du exactly (complex step, eps = 1e-30) on random 8x8 states."""
    nx = ny = 8
    eps = 1e-30
    m = _model(ora, dx=0.8, kappa_c=0.7, kappa_phi=1.3, W_c=1.9, W_phi=0.6)
    g = np.random.default_rng(7)
    c = g.random((ny, nx)); phi = g.random((ny, nx))
    mu_c, mu_p = ora.mu(m, c, phi)
    for field_idx, want in ((0, mu_c), (1, mu_p)):
        got = np.zeros((ny, nx))
        for j in range(ny):
            for i in range(nx):
                cc = c.astype(complex); pp = phi.astype(complex)
                (cc if field_idx == 0 else pp)[j, i] += 1j * eps
                got[j, i] = _energy_complex(m, cc, pp).imag / eps / m.dx**2
        np.testing.assert_allclose(want, got, atol=1e-13, rtol=0)
    # and the oracle's own energy diagnostic equals that energy
    assert ora.energy(m, c, phi) == pytest.approx(_energy_complex(m, c, phi).real, rel=1e-14)


def test_energy_cosine_mode_closed_form(ora):
    """c = 1/2 + a cos(2 pi m i/nx), phi = 1: E_h = dx^2 W_c N (1/16 - a^2/4 + 3a^4/8)
    + (kappa_c/2) a^2 ny nx (1 - cos(2 pi m/nx))."""
    nx, ny, a, mm = 64, 16, 0.2, 3
    m = _model(ora, dx=0.5, W_c=1.3, kappa_c=0.7, W_phi=2.0)
    c = inputs.cos_mode_x(nx, ny, mm, a)
    phi = np.ones((ny, nx))
    N = nx * ny
    want = m.dx**2 * m.W_c * N * (1 / 16 - a**2 / 4 + 3 * a**4 / 8) \
        + 0.5 * m.kappa_c * a**2 * ny * nx * (1 - math.cos(2 * math.pi * mm / nx))
    assert ora.energy(m, c, phi) == pytest.approx(want, rel=1e-14)
    d = ora.diagnostics(m, c, phi, np.zeros((ny, nx)))
    assert d[3] == pytest.approx(want, rel=1e-14)
    assert d[0] == pytest.approx(m.dx**2 * 0.5 * N, rel=1e-14)
    assert d[1] == pytest.approx(m.dx**2 * N, rel=1e-15)
    assert d[4] == 0


def test_nonfinite_count(ora):
    m = _model(ora)
    c, phi, rho = inputs.random_state(8, 8, 3)
    c[2, 3] = np.nan; phi[2, 3] = np.inf; rho[5, 5] = -np.inf
    assert ora.diagnostics(m, c, phi, rho)[4] == 2


# --------------------------------------------------------------------------- integrator
def _mode_amp_x(u, m_mode, base):
    nx = u.shape[1]
    cs = np.cos(2 * np.pi * m_mode * np.arange(nx) / nx)
    return 2.0 * ((u - base) * cs[None, :]).mean()


@pytest.mark.parametrize("mode,n", [(2, 1000), (5, 1000), (16, 100)])
def test_linear_growth_c_midpoint(ora, mode, n):
    """Small Fourier mode of c (phi = 1, v0 = 0, equal mobilities M):
    sigma = M lam (W_c - kappa_c lam), lam = (4/dx^2) sin^2(pi m/nx); per-step
    amplification G = 1 + sigma dt + (sigma dt)^2/2 (explicit midpoint)."""
    nx, ny, a = 64, 4, 1e-6
    M = 1.0
    m = _model(ora, dt=0.01, MA_bulk=M, MB_bulk=M, MA_surf=M, MB_surf=M, v_x=0.0, v_y=0.0)
    c = inputs.cos_mode_x(nx, ny, mode, a)
    phi = np.ones((ny, nx)); rho = np.ones((ny, nx))
    lam = 4 / m.dx**2 * math.sin(math.pi * mode / nx) ** 2
    sig = M * lam * (m.W_c - m.kappa_c * lam)
    G = 1 + sig * m.dt + (sig * m.dt) ** 2 / 2
    c1, _, _ = ora.step(m, c, phi, rho, n)
    want = a * G**n
    got = _mode_amp_x(c1, mode, 0.5)
    assert abs(got - want) <= 1e-8 * abs(want)
    # forward Euler is distinguishable under the same tolerance (unless the mode is ~neutral)
    ce, _, _ = ora.step(m, c, phi, rho, n, euler=True)
    ge = _mode_amp_x(ce, mode, 0.5)
    assert abs(ge - want) > 1e-7 * abs(want)


def test_linear_growth_phi_midpoint(ora):
    """Same for phi with c = 0 (c stays exactly 0): sigma = M_phi lam (W_phi - kappa_phi lam)."""
    nx, ny, a, n, mode = 64, 4, 1e-6, 1000, 3
    m = _model(ora, dt=0.01, M_phi=0.7, W_phi=1.5, kappa_phi=1.2, v_x=0.0, v_y=0.0)
    phi = inputs.cos_mode_x(nx, ny, mode, a)
    c = np.zeros((ny, nx)); rho = np.ones((ny, nx))
    lam = 4 / m.dx**2 * math.sin(math.pi * mode / nx) ** 2
    sig = m.M_phi * lam * (m.W_phi - m.kappa_phi * lam)
    G = 1 + sig * m.dt + (sig * m.dt) ** 2 / 2
    c1, p1, _ = ora.step(m, c, phi, rho, n)
    assert np.all(c1 == 0.0)
    got = _mode_amp_x(p1, mode, 0.5)
    assert abs(got - a * G**n) <= 1e-8 * abs(a * G**n)


def test_linear_growth_y_mode_no_flux(ora):
    """No-flux y boundary: cos(pi m (j+1/2)/ny) is an exact eigenvector of the mirror-rule L,
    lam = (4/dx^2) sin^2(pi m/(2 ny)); same growth law."""
    nx, ny, a, n, mode = 4, 48, 1e-6, 800, 4
    M = 1.0
    m = _model(ora, dt=0.01, MA_bulk=M, MB_bulk=M, MA_surf=M, MB_surf=M, v_x=0.0, v_y=0.0)
    c = inputs.cos_mode_y(nx, ny, mode, a)
    phi = np.ones((ny, nx)); rho = np.ones((ny, nx))
    lam = 4 / m.dx**2 * math.sin(math.pi * mode / (2 * ny)) ** 2
    sig = M * lam * (m.W_c - m.kappa_c * lam)
    G = 1 + sig * m.dt + (sig * m.dt) ** 2 / 2
    c1, _, _ = ora.step(m, c, phi, rho, n)
    cs = np.cos(np.pi * mode * (np.arange(ny) + 0.5) / ny)
    got = 2.0 * ((c1 - 0.5) * cs[:, None]).mean()
    assert abs(got - a * G**n) <= 1e-8 * abs(a * G**n)


def test_rho_reservoir_mode_decay(ora):
    """v0 = 0, phi uniform: rho = rho_in + a cos(k (j+1/2)), k = pi(q+1/2)/(ny+1/2), decays with
    sigma = -D_rho (4/dx^2) sin^2(k/2) (bottom mirror, top reservoir)."""
    nx, ny, q, a, n = 4, 32, 1, 0.1, 1500
    m = _model(ora, dt=0.01, D_rho=0.9, rho_in=0.6, v_x=0.0, v_y=0.0)
    k = math.pi * (q + 0.5) / (ny + 0.5)
    j = np.arange(ny)[:, None]
    rho = m.rho_in + a * np.cos(k * (j + 0.5)) * np.ones((1, nx))
    c = 0.5 * np.ones((ny, nx)); phi = 0.3 * np.ones((ny, nx))
    sig = -m.D_rho * 4 / m.dx**2 * math.sin(k / 2) ** 2
    G = 1 + sig * m.dt + (sig * m.dt) ** 2 / 2
    _, _, r1 = ora.step(m, c, phi, rho, n)
    want = m.rho_in + a * G**n * np.cos(k * (j + 0.5)) * np.ones((1, nx))
    assert np.max(np.abs(r1 - want)) <= 1e-10 * a


def test_rho_advection_mode(ora):
    """Central advection + diffusion (test-only theta = 0): product mode
    a cos(k(j+1/2)) Re(G^n e^{i 2 pi m i/nx}), z = dt(-D lam - i v_x sin(2 pi m/nx)/dx),
    lam = (4/dx^2)(sin^2(pi m/nx) + sin^2(k/2)), G = 1 + z + z^2/2."""
    nx, ny, q, mm, a, n = 32, 16, 0, 2, 0.05, 1000
    m = _model(ora, dt=0.01, D_rho=0.5, rho_in=1.0, v_x=0.8, v_y=-0.0)
    k = math.pi * (q + 0.5) / (ny + 0.5)
    j = np.arange(ny)[:, None]; i = np.arange(nx)[None, :]
    th = 2 * np.pi * mm * i / nx
    rho = m.rho_in + a * np.cos(k * (j + 0.5)) * np.cos(th)
    c = 0.5 * np.ones((ny, nx)); phi = np.ones((ny, nx))
    lam = 4 / m.dx**2 * (math.sin(math.pi * mm / nx) ** 2 + math.sin(k / 2) ** 2)
    z = m.dt * (-m.D_rho * lam - 1j * m.v_x * math.sin(2 * math.pi * mm / nx) / m.dx)
    G = 1 + z + z * z / 2
    _, _, r1 = ora.step(m, c, phi, rho, n)
    want = m.rho_in + a * np.cos(k * (j + 0.5)) * np.real(G**n * np.exp(1j * th))
    assert np.max(np.abs(r1 - want)) <= 1e-10 * a


# --------------------------------------------------------------------------- invariants
def test_uniform_state_is_fixed_point(ora):
    """Uniform c, phi and rho = rho_in: R == 0 exactly, state unchanged bit for bit."""
    m = _model(ora, v_x=0.1, v_y=-0.5, MA_bulk=2.0, MB_bulk=3.0)
    c = np.full((8, 16), 0.37); phi = np.full((8, 16), 0.81); rho = np.full((8, 16), m.rho_in)
    c1, p1, r1 = ora.step(m, c, phi, rho, 5)
    assert np.array_equal(c1, c) and np.array_equal(p1, phi) and np.array_equal(r1, rho)


def test_source_closed_form_and_bookkeeping(ora):
    """1-D tanh profile, theta = 90 deg, rho = 1: S = -v0 G_y phi (central difference,
    np.gradient in the interior).  S:255: sum R_phi = sum S because sum L(mu_phi) telescopes."""
    nx, ny, v0 = 8, 64, 0.7
    m = _model(ora, v_x=0.0, v_y=-v0)
    j = np.arange(ny)[:, None] * np.ones((1, nx))
    phi = 0.5 * (1 - np.tanh((j - 30.3) / 1.7))
    rho = np.ones((ny, nx))
    S = ora.source(m, phi, rho)
    want = -v0 * np.gradient(phi, axis=0)
    np.testing.assert_allclose(S[1:-1], want[1:-1], atol=1e-15)
    c, phi2, rho2 = inputs.random_state(16, 16, 11, phi_kind="smooth")
    m2 = _model(ora, v_x=0.2, v_y=-0.6)
    Rc, Rp, Rr, S2 = ora.rhs(m2, c, phi2, rho2)
    assert abs(Rp.sum() - S2.sum()) <= 1e-12 * np.abs(S2).sum()
    assert abs(Rc.sum()) <= 1e-12 * np.abs(Rc).sum()


def _vapour_boundary_sum(m, rho):
    """Sum over cells of D_rho L(rho) - v.G(rho) with the reservoir/mirror rules: everything
    telescopes except the top reservoir face and the y ends of the central difference."""
    dx = m.dx
    top, bot = rho[-1, :], rho[0, :]
    diff = m.D_rho * (m.rho_in - top) / dx**2
    adv = m.v_y * (m.rho_in + top - 2.0 * bot) / (2.0 * dx)
    return float(np.sum(diff - adv))


def test_vapour_sink_equals_paper_source_in_phit(ora):
    """P:331-340 in the paper's variable phit = 2 phi - 1 in [-1, 1]: the phit equation
    gains grad(phit).(rho v) and the rho equation loses exactly the same field.  With phi stored in
    [0, 1] (R-1) d(phit)/dt = 2 d(phi)/dt, so cell by cell
        2 (R_phi - M_phi L mu_phi) == -(R_rho - D_rho L rho + v.G rho) == rho v.G(phit).
    A sink of -S (half the paper's) fails this by a factor of 2."""
    nx = ny = 8
    for seed in range(3):
        g = np.random.default_rng(300 + seed)
        c = g.random((ny, nx)); phi = g.random((ny, nx)); rho = g.random((ny, nx))
        m = _model(ora, dx=0.7, M_phi=1.3, D_rho=0.6, rho_in=0.9, v_x=0.31, v_y=-0.57)
        Rc, Rp, Rr, S = ora.rhs(m, c, phi, rho)
        _, mu_p = ora.mu(m, c, phi)
        ch = m.M_phi * ora.laplacian(mu_p, m.dx)
        # the paper's phit source, written out with explicit neighbours (mirror rule in y, R-12)
        pt = 2.0 * phi - 1.0
        ptp = np.vstack([pt, pt[-1:]]); ptm = np.vstack([pt[:1], pt])
        gx = (np.roll(pt, -1, 1) - np.roll(pt, 1, 1)) / (2 * m.dx)
        gy = (ptp[1:] - ptm[:-1]) / (2 * m.dx)
        src_phit = rho * (m.v_x * gx + m.v_y * gy)
        rp = np.vstack([rho, np.full((1, nx), m.rho_in)]); rm = np.vstack([rho[:1], rho])
        lrho = (np.roll(rho, -1, 1) + np.roll(rho, 1, 1) + rp[1:] + rm[:-1] - 4 * rho) / m.dx**2
        vgr = m.v_x * (np.roll(rho, -1, 1) - np.roll(rho, 1, 1)) / (2 * m.dx) \
            + m.v_y * (rp[1:] - rm[:-1]) / (2 * m.dx)
        tol = 1e-13 * np.max(np.abs(src_phit))
        np.testing.assert_allclose(2.0 * (Rp - ch), src_phit, atol=tol, rtol=0)
        np.testing.assert_allclose(-(Rr - m.D_rho * lrho + vgr), src_phit, atol=tol, rtol=0)


def test_vapour_plus_solid_bookkeeping(ora):
    """P:331 + P:340: d/dt (phit + rho) is a pure divergence, so sum(rho + phit) = sum(rho + 2 phi)
    changes only through the boundary faces: per RHS, sum(R_rho + 2 R_phi) = B(rho) with B the top
    reservoir diffusion face and the y ends of the central advection; per midpoint step,
    sum(rho + 2 phi)^{n+1} - sum(rho + 2 phi)^n = dt B(rho*)."""
    c, phi, rho = inputs.random_state(16, 24, 17, phi_kind="smooth")
    m = _model(ora, nx=16, ny=24, D_rho=0.8, rho_in=0.9, v_x=0.2, v_y=-0.6)
    Rc, Rp, Rr, S = ora.rhs(m, c, phi, rho)
    B = _vapour_boundary_sum(m, rho)
    scale = np.abs(Rr).sum() + 2 * np.abs(Rp).sum()
    assert abs((Rr + 2 * Rp).sum() - B) <= 1e-13 * scale
    # a literal -S sink would leave sum(S) behind
    assert abs(S.sum()) > 1e-3 * scale
    # one step: u* from the RHS at u^n (P:348 midpoint), boundary sum at u*
    rs = rho + 0.5 * m.dt * Rr
    c1, p1, r1 = ora.step(m, c, phi, rho, 1)
    lhs = (r1 + 2 * p1).sum() - (rho + 2 * phi).sum()
    assert abs(lhs - m.dt * _vapour_boundary_sum(m, rs)) <= 1e-12 * m.dt * scale


def test_mass_conservation_with_and_without_source(ora):
    """c has no source: sum c is constant to round-off over 1000 steps, source on or off."""
    pr = ora.preset(1)
    c, phi, rho = ora.initial_fields(pr["ic"], 64, 64, 0)
    for vy in (-0.5, 0.0):
        m = _model(ora, v_x=0.0, v_y=vy)
        d0 = ora.diagnostics(m, c, phi, rho)
        c1, p1, r1 = ora.step(m, c, phi, rho, 1000)
        d1 = ora.diagnostics(m, c1, p1, r1)
        assert abs(d1[0] - d0[0]) <= 1e-12 * abs(d0[0])
        if vy == 0.0:  # and phi is conserved too without the source
            assert abs(d1[1] - d0[1]) <= 1e-12 * abs(d0[1])
        else:          # deposition grows the film
            assert d1[1] > d0[1]


def test_energy_monotone_decay_and_dissipation_identity(ora):
    """Pure Cahn-Hilliard (v0 = 0): E_h^{n+1} <= E_h^n every step; and the semi-discrete identity
    dE_h/dt = -sum_faces M_f (d mu_c)^2 - M_phi sum_faces (d mu_phi)^2 holds to O(dt)."""
    pr = ora.preset(1)
    c, phi, rho = ora.initial_fields(pr["ic"], 64, 64, 0)
    m = _model(ora, v_x=0.0, v_y=0.0)
    E = [ora.energy(m, c, phi)]
    for _ in range(200):
        c, phi, rho = ora.step(m, c, phi, rho, 1)
        E.append(ora.energy(m, c, phi))
    E = np.array(E)
    assert np.all(np.diff(E) <= 1e-14 * E[:-1])
    assert E[-1] < E[0]
    # dissipation identity at the current state
    D, ia, ib = _face_matrix(64, 64)
    mu_c, mu_p = ora.mu(m, c, phi)
    M = ora.mobility_field(m, c, phi).ravel()
    Mf = 0.5 * (M[ia] + M[ib])
    dmc = D @ mu_c.ravel(); dmp = D @ mu_p.ravel()
    rate = -(Mf * dmc**2).sum() - m.M_phi * (dmp**2).sum()
    errs = []
    for dt in (1e-3, 5e-4):
        mm = replace(m, dt=dt)
        c1, p1, _ = ora.step(mm, c, phi, rho, 1)
        fd = (ora.energy(mm, c1, p1) - ora.energy(mm, c, phi)) / dt
        errs.append(abs(fd - rate) / abs(rate))
    assert errs[0] < 1e-2
    assert errs[1] < 0.6 * errs[0]   # O(dt): halves with dt


def _relax_tanh(ora, dx, T):
    """Flat phi interface, c = 0, v0 = 0, kappa_phi = 1, W_phi = 1/8 (delta = 4 physical)."""
    Wp, kp = 1.0 / 8.0, 1.0
    delta = math.sqrt(2 * kp / Wp)
    L = 64.0
    ny = int(round(L / dx)); nx = 4
    m0 = _model(ora, dx=dx, W_phi=Wp, kappa_phi=kp, v_x=0.0, v_y=0.0)
    dt = 0.9 * ora.dt_max(m0, 1.0)
    m = replace(m0, dt=dt)
    y = (np.arange(ny) + 0.5) * dx
    y0 = L / 2
    prof = 0.5 * (1 - np.tanh((y - y0) / delta))
    phi = prof[:, None] * np.ones((1, nx))
    c = np.zeros((ny, nx)); rho = np.ones((ny, nx))
    n = int(round(T / dt))
    c1, p1, _ = ora.step(m, c, phi, rho, n)
    assert np.all(c1 == 0.0)
    return np.max(np.abs(p1[:, 0] - prof))


def test_tanh_equilibrium_profile(ora):
    """Flat interface relaxes to phi = 1/2 (1 - tanh((y - y0)/delta)), delta = sqrt(2 kappa/W),
    within O((dx/delta)^2): <= 5e-3 at delta/dx = 4."""
    err = _relax_tanh(ora, 1.0, 100.0)
    assert err <= 5e-3


@pytest.mark.slow
def test_tanh_equilibrium_second_order(ora):
    """Observed order >= 1.8 of the tanh deviation on dx halving."""
    e1 = _relax_tanh(ora, 1.0, 100.0)
    e2 = _relax_tanh(ora, 0.5, 100.0)
    assert math.log2(e1 / e2) >= 1.8


def test_stability_bound_values(ora):
    """R-18: dt_max = 1.6 / max(M_c (64 kappa_c/dx^4 + 16 W_c/dx^2), ...): 0.02 (cfg1), 2e-3 (cfg2-5)."""
    assert ora.dt_max(ora.preset(1)["model"], 1.0) == pytest.approx(0.02, rel=1e-15)
    assert ora.dt_max(ora.preset(2)["model"], 10.0) == pytest.approx(2e-3, rel=1e-15)


# --------------------------------------------------------------------------- regular solution (R-28)
def _energy_complex_rs(m, c, phi):
    """E_h with the regular-solution composition energy (R-28), complex-safe (no clamping: the
    states stay inside (1e-9, 1 - 1e-9))."""
    g = m.omega * c * (1 - c) + m.temp * (c * np.log(c) + (1 - c) * np.log(1 - c))
    f = g * phi + m.W_phi * phi**2 * (1 - phi) ** 2
    E = m.dx**2 * f.sum()
    for u, k in ((c, m.kappa_c), (phi, m.kappa_phi)):
        dxu = np.roll(u, -1, axis=1) - u
        dyu = u[1:, :] - u[:-1, :]
        E = E + 0.5 * k * ((dxu**2).sum() + (dyu**2).sum())
    return E


def test_regular_solution_mu_is_variational_derivative(ora):
    """R-28: mu = (1/dx^2) dE_h/du for the regular-solution energy (complex step)."""
    nx = ny = 6
    eps = 1e-30
    m = _model(ora, dx=0.9, kappa_c=0.6, kappa_phi=1.1, W_phi=0.8, fe=1, omega=2.7, temp=0.4)
    g = np.random.default_rng(11)
    c = 0.05 + 0.9 * g.random((ny, nx)); phi = g.random((ny, nx))
    mu_c, mu_p = ora.mu(m, c, phi)
    for field_idx, want in ((0, mu_c), (1, mu_p)):
        got = np.zeros((ny, nx))
        for j in range(ny):
            for i in range(nx):
                cc = c.astype(complex); pp = phi.astype(complex)
                (cc if field_idx == 0 else pp)[j, i] += 1j * eps
                got[j, i] = _energy_complex_rs(m, cc, pp).imag / eps / m.dx**2
        np.testing.assert_allclose(want, got, atol=1e-12, rtol=0)
    assert ora.energy(m, c, phi) == pytest.approx(_energy_complex_rs(m, c, phi).real, rel=1e-13)


@pytest.mark.parametrize("mode,n", [(3, 800), (6, 400), (20, 300)])
def test_regular_solution_linear_growth(ora, mode, n):
    """R-28 linearised about c = 1/2 (phi = 1, v0 = 0): g''(1/2) = -2 Omega + 4 T, so
    sigma = -M lam (g''(1/2) + kappa_c lam) and the midpoint factor G = 1 + sigma dt + (sigma dt)^2/2."""
    nx, ny, a = 64, 4, 1e-6
    M, Om, T = 1.0, 2.5, 0.5
    m = _model(ora, dt=0.01, MA_bulk=M, MB_bulk=M, MA_surf=M, MB_surf=M, v_x=0.0, v_y=0.0, fe=1, omega=Om, temp=T)
    c = inputs.cos_mode_x(nx, ny, mode, a)
    phi = np.ones((ny, nx)); rho = np.ones((ny, nx))
    lam = 4 / m.dx**2 * math.sin(math.pi * mode / nx) ** 2
    sig = -M * lam * ((-2 * Om + 4 * T) + m.kappa_c * lam)
    G = 1 + sig * m.dt + (sig * m.dt) ** 2 / 2
    c1, _, _ = ora.step(m, c, phi, rho, n)
    want = a * G**n
    assert abs(_mode_amp_x(c1, mode, 0.5) - want) <= 1e-8 * abs(want)


def test_regular_solution_energy_decay(ora):
    """Pure Cahn-Hilliard with the regular solution (v0 = 0): E_h non-increasing every step, c mass
    conserved."""
    m = _model(ora, dt=0.005, v_x=0.0, v_y=0.0, fe=1, omega=2.5, temp=0.5, W_phi=1.0)
    c, phi, rho = inputs.random_state(24, 20, 4, phi_kind="smooth")
    E = [ora.energy(m, c, phi)]
    mass0 = c.sum()
    for _ in range(60):
        c, phi, rho = ora.step(m, c, phi, rho, 1)
        E.append(ora.energy(m, c, phi))
    assert all(E[k + 1] <= E[k] + 1e-14 * abs(E[k]) for k in range(60))
    assert E[-1] < E[0]
    assert abs(c.sum() - mass0) <= 1e-12 * mass0
