"""Pins of the U-Net oracle (oracle/unet_oracle.py, NEXT-4) against things other than itself:
independent library routines (scipy correlate2d, torch.nn.functional), brute force on tiny inputs,
closed forms and exact identities of the paper's definitions (readings R-29..R-35)."""
import numpy as np
import pytest

from oracle import unet_oracle as U
from paper_2312_05410_b200 import synth


def _rng(s):
    return np.random.default_rng(s)


def test_conv_equals_scipy_correlate2d_same():
    from scipy.signal import correlate2d
    g = _rng(1)
    u = g.standard_normal((3, 7, 9))
    w = g.standard_normal((4, 3, 3, 3))
    got = U.conv(u, w)
    for o in range(4):
        want = sum(correlate2d(u[c], w[o, :, :, c], mode="same", boundary="fill") for c in range(3))
        assert np.allclose(got[o], want, rtol=0, atol=1e-12)


def test_conv_brute_force_tiny():
    g = _rng(2)
    u = g.standard_normal((2, 4, 5))
    w = g.standard_normal((3, 3, 3, 2))
    got = U.conv(u, w)
    for o in range(3):
        for i in range(4):
            for j in range(5):
                s = 0.0
                for k in range(2):
                    for m in range(3):
                        for n in range(3):
                            ii, jj = i + m - 1, j + n - 1
                            if 0 <= ii < 4 and 0 <= jj < 5:
                                s += u[k, ii, jj] * w[o, m, n, k]
                assert abs(got[o, i, j] - s) < 1e-13


def test_group_norm_matches_torch_and_moments():
    import torch
    g = _rng(3)
    u = 3.0 + 2.0 * g.standard_normal((8, 6, 5))
    gam, bet = g.standard_normal(8), g.standard_normal(8)
    got = U.group_norm(u, gam, bet, groups=4, eps=1e-5)
    want = torch.nn.functional.group_norm(torch.from_numpy(u[None]), 4, torch.from_numpy(gam),
                                          torch.from_numpy(bet), eps=1e-5)[0].numpy()
    assert np.allclose(got, want, rtol=0, atol=1e-12)
    # gamma = 1, beta = 0: every group has mean 0 and variance sigma^2 / (sigma^2 + eps)
    n = U.group_norm(u, np.ones(8), np.zeros(8), groups=4, eps=1e-5)
    for q in range(4):
        blk, raw = n[2 * q:2 * q + 2], u[2 * q:2 * q + 2]
        v = raw.var()
        assert abs(blk.mean()) < 1e-13
        assert abs(blk.var() - v / (v + 1e-5)) < 1e-12


def test_gelu_matches_torch_tanh_form_and_odd_identity():
    import torch
    x = np.linspace(-6, 6, 1001)
    want = torch.nn.functional.gelu(torch.from_numpy(x), approximate="tanh").numpy()
    assert np.allclose(U.gelu(x), want, rtol=0, atol=1e-14)
    assert np.allclose(U.gelu(x) - U.gelu(-x), x, rtol=0, atol=1e-13)   # 0.5x(1+t) + 0.5x(1-t) = x
    assert U.gelu(np.array([0.0]))[0] == 0.0


def test_down_matches_torch_maxpool():
    import torch
    u = _rng(4).standard_normal((3, 8, 6))
    want = torch.nn.functional.max_pool2d(torch.from_numpy(u[None]), 2, 2)[0].numpy()
    assert np.array_equal(U.down(u), want)


def test_up_is_depthwise_transposed_conv_and_adjoint_of_written_formula():
    import torch
    g = _rng(5)
    u = g.standard_normal((3, 4, 5))
    wt = g.standard_normal((2, 2))
    got = U.up(u, wt)
    k = torch.from_numpy(np.broadcast_to(wt, (3, 1, 2, 2)).copy())
    want = torch.nn.functional.conv_transpose2d(torch.from_numpy(u[None]), k, stride=2, groups=3)[0].numpy()
    assert np.allclose(got, want, rtol=0, atol=1e-14)
    # R-31: up is the adjoint of the formula as written in P:425, s(v)_{k,i,j} = sum v_{k,2i+m,2j+n} w_{m,n}
    v = g.standard_normal((3, 8, 10))
    s = sum(v[:, m::2, n::2] * wt[m, n] for m in range(2) for n in range(2))
    assert abs(np.sum(got * v) - np.sum(u * s)) < 1e-12


def test_time_basis_closed_forms():
    P = synth.unpack(synth.random_weights(7))
    Q = dict(P)
    Q["m_w0"] = np.zeros(128)
    assert np.array_equal(U.time_basis(0.3, Q), U.time_basis(4.0, Q))   # w0 = 0: constant in dt
    Q = dict(P)
    Q["m_w1"] = np.zeros((128, 128))
    Q["m_b1"] = np.full(128, np.pi / 2)
    Q["m_w2"] = np.eye(128)
    Q["m_b2"] = np.arange(128.0)
    assert np.allclose(U.time_basis(1.7, Q), 1.0 + np.arange(128.0), rtol=0, atol=1e-15)
    # one hidden unit, by hand: f = w2 sin(w1 sin(w0 dt + b0) + b1) + b2
    Q = {k: np.zeros_like(v) for k, v in P.items()}
    Q["m_w0"][0], Q["m_b0"][0] = 2.0, 0.1
    Q["m_w1"][5, 0], Q["m_b1"][5] = 1.5, -0.2
    Q["m_w2"][9, 5], Q["m_b2"][9] = 3.0, 0.25
    dt = 0.7
    f = U.time_basis(dt, Q)
    assert abs(f[9] - (3.0 * np.sin(1.5 * np.sin(2.0 * dt + 0.1) - 0.2) + 0.25)) < 1e-14
    assert np.count_nonzero(f) == 1


def _torch_forward(hist, dt, P):
    """The network composed from torch.nn.functional library ops (independent of the oracle)."""
    import torch
    F = torch.nn.functional
    T = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in P.items()}

    def cb(x, name, groups=8, act=True):   # R-30: min(8, C) = 8 for these widths
        w = T["w_" + name].permute(0, 3, 1, 2)          # [co, ci, 3, 3]
        y = F.group_norm(F.conv2d(x, w, padding=1), groups, T["g_" + name], T["b_" + name], eps=1e-5)
        return F.gelu(y, approximate="tanh") if act else y

    def upk(x, name):
        c = x.shape[1]
        return F.conv_transpose2d(x, T[name].expand(c, 1, 2, 2), stride=2, groups=c)

    x = torch.from_numpy(hist[None])
    h0 = torch.sin(T["m_w0"] * dt + T["m_b0"])
    f = T["m_w2"] @ torch.sin(T["m_w1"] @ h0 + T["m_b1"]) + T["m_b2"]
    z1 = cb(x, "enc1")
    z2 = cb(F.max_pool2d(z1, 2), "enc2")
    z3 = cb(F.max_pool2d(z2, 2), "enc3")
    z4 = cb(F.max_pool2d(z3, 2), "enc4")
    zc = [z * (T[f"wl{p}"] @ f)[None, :, None, None] for p, z in enumerate((z1, z2, z3, z4), 1)]
    d3 = upk(cb(zc[3], "dec4"), "up3")
    d2 = upk(cb(torch.cat([zc[2], d3], 1), "dec3"), "up2")
    d1 = upk(cb(torch.cat([zc[1], d2], 1), "dec2"), "up1")
    h = cb(torch.cat([zc[0], d1], 1), "head1")
    return cb(h, "head2", groups=1, act=False)[0, 0].numpy()


@pytest.mark.parametrize("hw", [(16, 16), (32, 24)])
def test_forward_matches_torch_functional_composition(hw):
    H, W = hw
    P = synth.unpack(synth.random_weights(11))
    hist = synth.histories(1, 3, H, W, seed=12)[0]
    got = U.forward(hist, 2.0, P)
    want = _torch_forward(hist, 2.0, P)
    assert got.shape == (H, W)
    assert np.allclose(got, want, rtol=0, atol=1e-10)


def test_forward_shape_contract_levels_and_degeneracies():
    P = synth.unpack(synth.random_weights(13))
    hist = synth.histories(2, 3, 32, 32, seed=14)
    z = U.encode(hist[0], P)
    assert [t.shape for t in z] == [(16, 32, 32), (32, 16, 16), (64, 8, 8), (128, 4, 4)]
    # z^{L2} = conv_block(down(z^{L1})) by hand composition
    assert np.array_equal(z[1], U.conv_block(U.down(z[0]), P["w_enc2"], P["g_enc2"], P["b_enc2"]))
    # w0 = 0 => forward independent of dt
    Q = dict(P)
    Q["m_w0"] = np.zeros(128)
    assert np.array_equal(U.forward(hist[0], 1.0, Q), U.forward(hist[0], 5.0, Q))
    # the dt conditioning does act when w0 != 0
    assert not np.allclose(U.forward(hist[0], 1.0, P), U.forward(hist[0], 2.0, P))
    # all-ones conditioning (f = e_0, w^{Lp}[:, 0] = 1) leaves the latents unchanged
    Q = dict(P)
    Q["m_w2"], Q["m_b2"] = np.zeros((128, 128)), np.eye(128)[0]
    for p, c in enumerate((16, 32, 64, 128), 1):
        Q[f"wl{p}"] = np.zeros((c, 128))
        Q[f"wl{p}"][:, 0] = 1.0
    zc = U.condition(z, 3.0, Q)
    assert all(np.array_equal(a, b) for a, b in zip(zc, z))
    # batch: per-sample independence
    out = U.forward_batch(hist, [1.0, 2.0], P)
    assert np.array_equal(out[1], U.forward(hist[1], 2.0, P))
