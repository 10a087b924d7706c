"""ctypes binding of the CPU oracle (oracle/pf_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg.  The product package
(paper_2312_05410_b200) never imports this module and shares no code with it.

The presets below are the oracle's own copy of the workload parameters
(readings R-13/R-14, from SURVEY.md 8(c.2) and
BASELINE.json configs[0..4]); tests check that the library's
``pf_default_params`` agrees with them rather than feeding library values into
the oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field, asdict

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle: plain C, -O2, no FMA contraction, no fast-math (R-16, R-19)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Model(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("dx", C.c_double), ("dt", C.c_double),
                ("kappa_c", C.c_double), ("kappa_phi", C.c_double), ("W_c", C.c_double),
                ("W_phi", C.c_double), ("MA_bulk", C.c_double), ("MB_bulk", C.c_double),
                ("MA_surf", C.c_double), ("MB_surf", C.c_double), ("sigma_surf", C.c_double),
                ("M_phi", C.c_double), ("D_rho", C.c_double), ("rho_in", C.c_double),
                ("v_x", C.c_double), ("v_y", C.c_double), ("fe", C.c_int32), ("omega", C.c_double),
                ("temp", C.c_double)]


class _IC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("height", C.c_double), ("amp", C.c_double),
                ("wavelength", C.c_double), ("ncols", C.c_int32), ("c0", C.c_double),
                ("c_lo", C.c_double), ("c_hi", C.c_double), ("noise_c", C.c_double),
                ("noise_phi", C.c_double), ("noise_c_gaussian", C.c_int32),
                ("kappa_phi", C.c_double), ("W_phi", C.c_double), ("rho_in", C.c_double),
                ("v0", C.c_double), ("theta_deg", C.c_double), ("rate_lo", C.c_double),
                ("rate_hi", C.c_double), ("theta_span", C.c_double), ("mob_lo", C.c_double),
                ("mob_hi", C.c_double), ("seed", C.c_uint64)]


IC_KINDS = {"film": 0, "rough": 1, "columns": 2}


@dataclass
class Model:
    """Physical/numerical parameters of one member."""
    nx: int = 64
    ny: int = 64
    dx: float = 1.0
    dt: float = 1e-3
    kappa_c: float = 1.0
    kappa_phi: float = 1.0
    W_c: float = 1.0
    W_phi: float = 1.0
    MA_bulk: float = 1.0
    MB_bulk: float = 1.0
    MA_surf: float = 1.0
    MB_surf: float = 1.0
    sigma_surf: float = 0.5
    M_phi: float = 1.0
    D_rho: float = 1.0
    rho_in: float = 1.0
    v_x: float = 0.0
    v_y: float = 0.0
    fe: int = 0            # 0 polynomial composition well (R-2), 1 regular solution (R-28)
    omega: float = 0.0
    temp: float = 0.0

    def _c(self, shape=None) -> _Model:
        d = {k: getattr(self, k) for k, _ in _Model._fields_}
        if shape is not None:          # the arrays decide the grid size
            d["ny"], d["nx"] = int(shape[0]), int(shape[1])
        return _Model(**d)


@dataclass
class IC:
    """Initial-condition recipe (R-14) plus the deposition sweep (R-15)."""
    kind: str = "film"
    height: float = 16.0
    amp: float = 0.0
    wavelength: float = 32.0
    ncols: int = 0
    c0: float = 0.5
    c_lo: float = 0.2
    c_hi: float = 0.8
    noise_c: float = 0.05
    noise_phi: float = 0.01
    noise_c_gaussian: bool = False
    kappa_phi: float = 1.0
    W_phi: float = 1.0
    rho_in: float = 1.0
    v0: float = 0.5
    theta_deg: float = 90.0
    rate_lo: float = 1.0
    rate_hi: float = 1.0
    theta_span: float = 0.0
    mob_lo: float = 1.0
    mob_hi: float = 1.0
    seed: int = 1

    def _c(self) -> _IC:
        d = asdict(self)
        d["kind"] = IC_KINDS[self.kind]
        d["noise_c_gaussian"] = int(self.noise_c_gaussian)
        return _IC(**d)


# --------------------------------------------------------------------------- presets
# The oracle's own copy of the five BASELINE workloads (R-13, R-14, R-15).
def preset(cfg: int) -> dict:
    """Return {'model': Model, 'ic': IC, 'members': int, 'steps': int, 'precision': str}."""
    if cfg == 1:
        m = Model(nx=64, ny=64)
        ic = IC(kind="film", height=16.0, c0=0.5, noise_c=0.05, noise_phi=0.01, seed=1)
        return dict(model=m, ic=ic, members=1, steps=1000, precision="f64")
    mob = dict(MA_bulk=10.0, MB_bulk=10.0, MA_surf=10.0, MB_surf=10.0, M_phi=1.0)
    if cfg == 2:
        m = Model(nx=256, ny=256, **mob)
        ic = IC(kind="rough", height=32.0, amp=2.0, wavelength=32.0, noise_c=0.05,
                noise_phi=0.0, noise_c_gaussian=True, seed=2)
        return dict(model=m, ic=ic, members=1, steps=10000, precision="f64")
    if cfg == 3:
        m = Model(nx=512, ny=512, **mob)
        ic = IC(kind="rough", height=32.0, amp=2.0, wavelength=32.0, noise_c=0.05,
                noise_phi=0.0, noise_c_gaussian=True, rate_lo=0.5, rate_hi=2.0, seed=3)
        return dict(model=m, ic=ic, members=64, steps=5000, precision="f64")
    if cfg == 4:
        m = Model(nx=4096, ny=4096, **mob)
        ic = IC(kind="rough", height=512.0, amp=2.0, wavelength=32.0, noise_c=0.05,
                noise_phi=0.0, noise_c_gaussian=True, seed=4)
        return dict(model=m, ic=ic, members=1, steps=2000, precision="f64")
    if cfg == 5:
        m = Model(nx=8192, ny=8192, **mob)
        ic = IC(kind="columns", height=4096.0, amp=0.0, ncols=64, c_lo=0.2, c_hi=0.8,
                noise_c=0.0, noise_phi=0.0, seed=5)
        return dict(model=m, ic=ic, members=1, steps=1000, precision="f32")
    raise ValueError(f"no preset {cfg}")


# --------------------------------------------------------------------------- library
_lib = None
_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dbl, i32, i64, u64 = C.c_double, C.c_int32, C.c_int64, C.c_uint64
        pM, pI = C.POINTER(_Model), C.POINTER(_IC)
        sig = {
            "orc_h": (dbl, [dbl]), "orc_p": (dbl, [dbl]), "orc_e": (dbl, [dbl, dbl]),
            "orc_mobility_c": (dbl, [pM, dbl, dbl]),
            "orc_laplacian": (None, [C.c_int, C.c_int, dbl, _D, C.c_int, dbl, _D]),
            "orc_gradient": (None, [C.c_int, C.c_int, dbl, _D, C.c_int, dbl, _D, _D]),
            "orc_mu": (None, [pM, _D, _D, _D, _D]),
            "orc_mobility_field": (None, [pM, _D, _D, _D]),
            "orc_source": (None, [pM, _D, _D, _D]),
            "orc_rhs": (None, [pM, _D, _D, _D, _D, _D, _D, _D]),
            "orc_step": (None, [pM, _D, _D, _D]),
            "orc_step_euler": (None, [pM, _D, _D, _D]),
            "orc_run": (None, [pM, _D, _D, _D, i64]),
            "orc_energy": (dbl, [pM, _D, _D]),
            "orc_diagnostics": (None, [pM, _D, _D, _D, _D]),
            "orc_sm64": (u64, [u64]), "orc_draw": (u64, [u64, u64, u64]),
            "orc_uniform": (dbl, [u64, u64, u64]), "orc_gauss": (dbl, [u64, u64, u64]),
            "orc_member_velocity": (None, [pI, i64, C.POINTER(dbl), C.POINTER(dbl)]),
            "orc_member_mobility": (None, [pI, i64, C.POINTER(dbl), C.POINTER(dbl)]),
            "orc_inflow": (dbl, [C.c_uint64, i64, i64, C.c_int, C.c_int, dbl, dbl]),
            "orc_run_inflow": (None, [pM, _D, _D, _D, i64, i64, C.c_uint64, i64, dbl]),
            "orc_initial_fields": (C.c_int, [pI, C.c_int, C.c_int, i64, _D, _D, _D]),
            "orc_initial_fields_rows": (C.c_int, [pI, C.c_int, i64, C.c_int, C.c_int, _D, _D, _D]),
            "orc_dt_max": (dbl, [pM, dbl]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


MIRROR, RESERVOIR = 0, 1


def _a(x):
    return np.ascontiguousarray(x, dtype=np.float64)


# Pointwise functions ----------------------------------------------------------------
def h(c): return lib().orc_h(float(c))
def p(phi): return lib().orc_p(float(phi))
def e(phi, sigma): return lib().orc_e(float(phi), float(sigma))
def mobility_c(m: Model, c, phi): return lib().orc_mobility_c(C.byref(m._c()), float(c), float(phi))


# Field operators ----------------------------------------------------------------------
def laplacian(u, dx=1.0, rule=MIRROR, top=0.0):
    u = _a(u); out = np.empty_like(u)
    lib().orc_laplacian(u.shape[1], u.shape[0], dx, u, rule, top, out)
    return out


def gradient(u, dx=1.0, rule=MIRROR, top=0.0):
    u = _a(u); gx = np.empty_like(u); gy = np.empty_like(u)
    lib().orc_gradient(u.shape[1], u.shape[0], dx, u, rule, top, gx, gy)
    return gx, gy


def mu(m: Model, c, phi):
    c, phi = _a(c), _a(phi); a = np.empty_like(c); b = np.empty_like(c)
    lib().orc_mu(C.byref(m._c(c.shape)), c, phi, a, b)
    return a, b


def mobility_field(m: Model, c, phi):
    c, phi = _a(c), _a(phi); M = np.empty_like(c)
    lib().orc_mobility_field(C.byref(m._c(c.shape)), c, phi, M)
    return M


def source(m: Model, phi, rho):
    phi, rho = _a(phi), _a(rho); S = np.empty_like(phi)
    lib().orc_source(C.byref(m._c(phi.shape)), phi, rho, S)
    return S


def rhs(m: Model, c, phi, rho):
    """Return (R_c, R_phi, R_rho, S)."""
    c, phi, rho = _a(c), _a(phi), _a(rho)
    assert c.shape == phi.shape == rho.shape
    out = [np.empty_like(c) for _ in range(4)]
    lib().orc_rhs(C.byref(m._c(c.shape)), c, phi, rho, *out)
    return tuple(out)


def step(m: Model, c, phi, rho, n: int = 1, euler: bool = False):
    """Advance copies of (c, phi, rho) by n explicit-midpoint steps (or Euler)."""
    c, phi, rho = _a(c).copy(), _a(phi).copy(), _a(rho).copy()
    assert c.shape == phi.shape == rho.shape
    mc = m._c(c.shape)
    if euler:
        for _ in range(n):
            lib().orc_step_euler(C.byref(mc), c, phi, rho)
    else:
        lib().orc_run(C.byref(mc), c, phi, rho, int(n))
    return c, phi, rho


def inflow(seed: int, member: int, step: int, nx: int, i: int, rho_in: float, sigma: float) -> float:
    """Stochastic reservoir value of column i at global step `step` (R-27)."""
    return lib().orc_inflow(seed, member, step, nx, i, rho_in, sigma)


def step_inflow(m: Model, c, phi, rho, n: int, step0: int, seed: int, member: int, sigma: float):
    """n midpoint steps with the per-step stochastic inflow row (R-27); step0 = global step index."""
    c, phi, rho = _a(c).copy(), _a(phi).copy(), _a(rho).copy()
    lib().orc_run_inflow(C.byref(m._c(c.shape)), c, phi, rho, int(n), int(step0), seed, int(member), float(sigma))
    return c, phi, rho


def energy(m: Model, c, phi):
    c, phi = _a(c), _a(phi)
    assert c.shape == phi.shape
    return lib().orc_energy(C.byref(m._c(c.shape)), c, phi)


def diagnostics(m: Model, c, phi, rho):
    out = np.zeros(5)
    c, phi, rho = _a(c), _a(phi), _a(rho)
    assert c.shape == phi.shape == rho.shape
    lib().orc_diagnostics(C.byref(m._c(c.shape)), c, phi, rho, out)
    return out


def dt_max(m: Model, M_c_max: float):
    return lib().orc_dt_max(C.byref(m._c()), float(M_c_max))


# RNG and initial conditions ---------------------------------------------------------
def sm64(z): return lib().orc_sm64(z)
def draw(seed, stream, k): return lib().orc_draw(seed, stream, k)
def uniform(seed, stream, k): return lib().orc_uniform(seed, stream, k)
def gauss(seed, stream, idx): return lib().orc_gauss(seed, stream, idx)


def member_velocity(ic: IC, member: int):
    vx, vy = C.c_double(), C.c_double()
    lib().orc_member_velocity(C.byref(ic._c()), int(member), C.byref(vx), C.byref(vy))
    return vx.value, vy.value


def initial_fields(ic: IC, nx: int, ny: int, member: int = 0):
    c = np.empty((ny, nx)); phi = np.empty((ny, nx)); rho = np.empty((ny, nx))
    rc = lib().orc_initial_fields(C.byref(ic._c()), nx, ny, int(member), c, phi, rho)
    if rc != 0:
        raise ValueError("bad IC recipe")
    return c, phi, rho


def initial_fields_rows(ic: IC, nx: int, member: int, y0: int, rows: int):
    """Global rows [y0, y0+rows) of the member's initial fields (same values as the full grid)."""
    c = np.empty((rows, nx)); phi = np.empty((rows, nx)); rho = np.empty((rows, nx))
    rc = lib().orc_initial_fields_rows(C.byref(ic._c()), nx, int(member), int(y0), int(rows), c, phi, rho)
    if rc != 0:
        raise ValueError("bad IC recipe")
    return c, phi, rho


def member_mobility(ic: IC, member: int):
    """(a, b): multipliers of the species-A and species-B mobilities of global member (R-23)."""
    a, b = C.c_double(), C.c_double()
    lib().orc_member_mobility(C.byref(ic._c()), int(member), C.byref(a), C.byref(b))
    return a.value, b.value


def member_model_sweep(m: Model, ic: IC, member: int) -> Model:
    """Copy of Model m with member's velocity (R-10, R-15, R-21) and mobilities (R-23)."""
    q = Model(**asdict(m))
    q.v_x, q.v_y = member_velocity(ic, member)
    a, b = member_mobility(ic, member)
    q.MA_bulk, q.MA_surf = m.MA_bulk * a, m.MA_surf * a
    q.MB_bulk, q.MB_surf = m.MB_bulk * b, m.MB_surf * b
    return q


def composite(c, phi):
    """Composite composition field of a dataset snapshot ("50 time snapshots"; SPEC S:442:
    the stored field carries c in the solid and exactly 0 in the vapour): c where phi > 1/2."""
    c, phi = np.asarray(c, dtype=np.float64), np.asarray(phi, dtype=np.float64)
    return np.where(phi > 0.5, c, 0.0)


def member_model(cfg_or_preset, member: int) -> Model:
    """Model of global member `member` with its own velocity (R-15)."""
    pr = preset(cfg_or_preset) if isinstance(cfg_or_preset, int) else cfg_or_preset
    m = Model(**asdict(pr["model"]))
    m.v_x, m.v_y = member_velocity(pr["ic"], member)
    return m


# --------------------------------------------------------------------------- NEXT-2 statistics
# Microstructure statistics of the paper's evaluation (section 2.3, P:486-504 section
# 4.5; SPEC S:456-526 and readings R-24..R-26 of DESIGN.md 11).  numpy, fp64; the FFT is a
# library primitive used as one step of the stated definition.

def indicator(comp, threshold=0.5):
    """Phase-A indicator of a composite field (R-24): 1 where c >= threshold (the vapour carries
    c = 0 in the composite, so it is never phase A), else 0."""
    return (np.asarray(comp, dtype=np.float64) >= threshold).astype(np.float64)


def s2_direct(ind):
    """S2(r) = (1/N) sum_x I(x) I(x + r), periodic, N = number of cells, by the double sum
    (brute force, small grids only); returned centered: out[ny//2 + dy, nx//2 + dx]."""
    I = np.asarray(ind, dtype=np.float64)
    ny, nx = I.shape
    out = np.zeros((ny, nx))
    for dy in range(-(ny // 2), ny - ny // 2):
        for dx in range(-(nx // 2), nx - nx // 2):
            acc = 0.0
            for y in range(ny):
                for x in range(nx):
                    acc += I[y, x] * I[(y + dy) % ny, (x + dx) % nx]
            out[ny // 2 + dy, nx // 2 + dx] = acc / (nx * ny)
    return out


def s2_fft(ind):
    """Same as s2_direct through the Wiener-Khinchin identity: ifft(|fft(I)|^2) / N, centered."""
    I = np.asarray(ind, dtype=np.float64)
    F = np.fft.fft2(I)
    corr = np.real(np.fft.ifft2(F * np.conj(F))) / I.size
    return np.fft.fftshift(corr)


def radial_bins(ny, nx):
    """Bin of every entry of a centered map: round(|r|) (R-25, integer-radius bins)."""
    dy = np.arange(ny)[:, None] - ny // 2
    dx = np.arange(nx)[None, :] - nx // 2
    return np.floor(np.sqrt(dx * dx + dy * dy) + 0.5).astype(np.int64)


def radial_average(s2):
    """Mean of the centered map over each integer-radius bin; bins 0 .. max."""
    b = radial_bins(*s2.shape)
    n = b.max() + 1
    sums = np.bincount(b.ravel(), weights=np.asarray(s2, dtype=np.float64).ravel(), minlength=n)
    cnt = np.bincount(b.ravel(), minlength=n)
    return sums / cnt


def rel_l2(true, pred):
    """Rel. L2 = ||true - pred||_2 / ||true||_2."""
    t, p = np.asarray(true, dtype=np.float64), np.asarray(pred, dtype=np.float64)
    return float(np.sqrt(np.sum((t - p) ** 2)) / np.sqrt(np.sum(t ** 2)))


def rel_mse(true, pred):
    """Rel. MSE in the norm-ratio reading (R-26): sum (t - p)^2 / sum t^2."""
    t, p = np.asarray(true, dtype=np.float64), np.asarray(pred, dtype=np.float64)
    return float(np.sum((t - p) ** 2) / np.sum(t ** 2))
