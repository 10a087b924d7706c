"""Pins of the oracle's NEXT-2 statistics (S2 autocorrelation, radial average, Rel. L2 / MSE;
P:196-206): closed forms and brute force, no GPU."""
import numpy as np
import pytest


def test_s2_closed_forms(ora):
    N = 12
    ones = np.ones((N, N))
    assert np.allclose(ora.s2_direct(ones), 1.0) and np.allclose(ora.s2_fft(ones), 1.0, atol=1e-15)
    assert np.array_equal(ora.s2_direct(np.zeros((N, N))), np.zeros((N, N)))
    one = np.zeros((N, N)); one[3, 7] = 1.0
    s = ora.s2_direct(one)
    assert s[N // 2, N // 2] == 1.0 / N ** 2 and np.count_nonzero(s) == 1
    # stripes of period 2 along x: S2(dx, dy) = 1/2 for even dx, 0 for odd dx
    st = np.zeros((8, 10)); st[:, ::2] = 1.0
    s = ora.s2_direct(st)
    dx = np.arange(10)[None, :] - 5
    assert np.array_equal(s, np.where(dx % 2 == 0, 0.5, 0.0) * np.ones((8, 1)))


def test_s2_fft_equals_direct_and_invariants(ora):
    """The FFT form equals the brute-force double sum on random 16 x 16 indicators (1e-12 abs);
    S2(0) = volume fraction; symmetry under r -> -r; 0 <= S2 <= S2(0)."""
    g = np.random.default_rng(5)
    for _ in range(3):
        I = (g.random((16, 16)) < 0.4).astype(float)
        a, b = ora.s2_direct(I), ora.s2_fft(I)
        assert np.abs(a - b).max() < 1e-12
        assert a[8, 8] == I.mean()
        assert np.array_equal(a[1:, 1:], a[1:, 1:][::-1, ::-1])   # r -> -r about the center
        assert a.min() >= 0 and a.max() <= a[8, 8] + 1e-15


def test_radial_average_pins(ora):
    s = np.full((16, 16), 0.3)
    assert np.allclose(ora.radial_average(s), 0.3)
    I = (np.random.default_rng(1).random((16, 16)) < 0.5).astype(float)
    m = ora.s2_direct(I)
    r = ora.radial_average(m)
    assert r[0] == m[8, 8]
    # isotropic map exp(-|r|): each bin's mean is within one bin width of exp(-bin)
    dy = np.arange(32)[:, None] - 16
    dx = np.arange(32)[None, :] - 16
    iso = np.exp(-np.sqrt(dx * dx + dy * dy))
    prof = ora.radial_average(iso)
    for k in range(1, 12):
        assert np.exp(-(k + 0.5)) - 1e-15 <= prof[k] <= np.exp(-(k - 0.5)) + 1e-15


def test_error_metrics(ora):
    g = np.random.default_rng(2)
    t = g.random((9, 7))
    assert ora.rel_l2(t, t) == 0.0 and ora.rel_l2(t, 0 * t) == 1.0
    assert ora.rel_l2(t, 1.25 * t) == pytest.approx(0.25, rel=1e-14)
    assert ora.rel_mse(t, 0 * t) == 1.0 and ora.rel_mse(t, 2 * t) == pytest.approx(1.0, rel=1e-14)
    assert np.array_equal(ora.indicator(np.array([0.0, 0.49, 0.5, 0.9])), np.array([0.0, 0.0, 1.0, 1.0]))
