"""Seeded synthetic inputs shared by the oracle tests and the GPU parity tests.

This module holds NO arithmetic of the method (no chemical potential, mobility,
flux, source or update): only numpy random draws and simple analytic profiles
used as test inputs.  Both sides receive the same arrays.
"""
import numpy as np


def random_state(nx, ny, seed, *, c_amp=0.05, phi_kind="film", height=None, rho_in=1.0):
    """(c, phi, rho) with c ~ 0.5 + U(-c_amp, c_amp), phi a noisy film or uniform noise."""
    g = np.random.default_rng(seed)
    c = 0.5 + c_amp * (2 * g.random((ny, nx)) - 1)
    if phi_kind == "film":
        H = ny // 4 if height is None else height
        base = (np.arange(ny)[:, None] < H).astype(float) * np.ones((1, nx))
        phi = base + 0.01 * (2 * g.random((ny, nx)) - 1)
        rho = rho_in * (1 - base)
    elif phi_kind == "noise":
        phi = g.random((ny, nx))
        rho = rho_in * g.random((ny, nx))
    elif phi_kind == "smooth":
        y = np.arange(ny)[:, None] + 0.0 * np.arange(nx)[None, :]
        x = np.arange(nx)[None, :] + 0.0 * y
        H = ny / 3 + 2 * np.sin(2 * np.pi * x / max(nx, 1))
        phi = 0.5 * (1 - np.tanh((y - H) / 1.5)) + 0.01 * (2 * g.random((ny, nx)) - 1)
        rho = rho_in * (1 - phi) + 0.01 * g.random((ny, nx))
    else:
        raise ValueError(phi_kind)
    return c, phi, rho


def cos_mode_x(nx, ny, m, a, base=0.5):
    i = np.arange(nx)[None, :]
    return base + a * np.cos(2 * np.pi * m * i / nx) * np.ones((ny, 1))


def cos_mode_y(nx, ny, m, a, base=0.5):
    j = np.arange(ny)[:, None]
    return base + a * np.cos(np.pi * m * (j + 0.5) / ny) * np.ones((1, nx))
