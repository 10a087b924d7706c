"""CPU oracle of the temporally conditioned U-Net, float64, numpy.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs.  The product package never imports it and shares no code
with it; the weights and histories it receives come from paper_2312_05410_b200/synth.py (seeded
draws, no arithmetic of the method).

Every function follows the paper's definition in its order and notation (P = PAPER.md line):
  conv        P:383-387  conv(u)_{k',i,j} = sum_k sum_m sum_n u_{k,i+m,j+n} w_{k,k',m,n}
              read as a 3x3 'same' cross-correlation with one zero cell of padding (R-29)
  group_norm  P:389-405  mu_g, sigma_g^2 over (C/G channels x W x H), (u - mu)/sqrt(sigma^2 + eps),
              then gamma_k u_hat + beta_k (R-30: G = min(8, C) = 8 groups, eps = 1e-5)
  gelu        P:408-411  0.5 u (1 + tanh(sqrt(2/pi) (u + 0.044715 u^3)))
  conv_block  P:412-415  GELU(GN(conv(u)))
  down        P:417-422  2x2 max pooling, stride 2
  up          P:423-428  up(u)_{k, 2i+m, 2j+n} = u_{k,i,j} w^{tconv}_{m,n}: the transpose of the
              written (garbled, subsampling) formula, one 2x2 kernel per up operation (R-31)
  time_basis  P:367-372  f(dt) = w2 sin(w1 sin(w0 dt + b0) + b1) + b2
  forward     P:431-462  encoder z^{L1..L4}, conditioning z (.) (w^{Lp} f(dt)), decoder d^{L3..L1},
              output GN(conv(conv_block(z^{L1} (+) d^{L1})))  (R-32..R-35)
A library primitive (numpy einsum / tensordot) serves as the channel contraction of conv and the
matrix-vector products of the MLP.
"""
from __future__ import annotations

import numpy as np

GROUPS = 8       # R-30: G = min(8, C) (SPEC), 8 for every width used (16 .. 128)
EPS = 1e-5       # R-30


def conv(u, w):
    """u [C, H, W], w [C', 3, 3, C] -> [C', H, W]; zero padding of one cell (R-29)."""
    C, H, W = u.shape
    up_ = np.zeros((C, H + 2, W + 2))
    up_[:, 1:H + 1, 1:W + 1] = u
    out = np.zeros((w.shape[0], H, W))
    for m in range(3):            # m: row offset (i + m - 1), n: column offset (j + n - 1)
        for n in range(3):
            out += np.einsum("oc,chw->ohw", w[:, m, n, :], up_[:, m:m + H, n:n + W])
    return out


def group_norm(u, gamma, beta, groups=GROUPS, eps=EPS):
    C, H, W = u.shape
    Ct = C // groups
    out = np.empty_like(u)
    for g in range(groups):
        blk = u[g * Ct:(g + 1) * Ct]
        mu = blk.sum() / (Ct * W * H)
        var = ((blk - mu) ** 2).sum() / (Ct * W * H)
        out[g * Ct:(g + 1) * Ct] = (blk - mu) / np.sqrt(var + eps)
    return gamma[:, None, None] * out + beta[:, None, None]


def gelu(u):
    return 0.5 * u * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (u + 0.044715 * u ** 3)))


def conv_block(u, w, gamma, beta, groups=GROUPS):
    return gelu(group_norm(conv(u, w), gamma, beta, groups))


def down(u):
    C, H, W = u.shape
    return u.reshape(C, H // 2, 2, W // 2, 2).max(axis=(2, 4))


def up(u, wt):
    C, H, W = u.shape
    out = np.empty((C, 2 * H, 2 * W))
    for m in range(2):
        for n in range(2):
            out[:, m::2, n::2] = u * wt[m, n]
    return out


def time_basis(dt, P):
    h0 = np.sin(P["m_w0"] * dt + P["m_b0"])
    h1 = np.sin(P["m_w1"] @ h0 + P["m_b1"])
    return P["m_w2"] @ h1 + P["m_b2"]


def groups_of(c):
    """Group count of a C-channel GroupNorm (R-30, SPEC): G = min(8, C), or G = C when C is not a
    multiple of it (the 1-channel output: G = 1)."""
    g = min(GROUPS, c)
    return g if c % g == 0 else c


def encode(hist, P):
    """z^{L1..L4}_t."""
    z = []
    for p, name in enumerate(("enc1", "enc2", "enc3", "enc4")):
        x = hist if p == 0 else down(z[-1])
        z.append(conv_block(x, P["w_" + name], P["g_" + name], P["b_" + name]))
    return z


def condition(z, dt, P):
    """z^{Lp}_{t+dt} = z^{Lp}_t (.) w^{Lp} f(dt)."""
    f = time_basis(dt, P)
    return [zp * (P[f"wl{p + 1}"] @ f)[:, None, None] for p, zp in enumerate(z)]


def decode(zc, P):
    """d^{L3}, d^{L2}, d^{L1} and the output."""
    cb = lambda x, name: conv_block(x, P["w_" + name], P["g_" + name], P["b_" + name])
    d3 = up(cb(zc[3], "dec4"), P["up3"])
    d2 = up(cb(np.concatenate([zc[2], d3]), "dec3"), P["up2"])
    d1 = up(cb(np.concatenate([zc[1], d2]), "dec2"), P["up1"])
    h = cb(np.concatenate([zc[0], d1]), "head1")
    out = group_norm(conv(h, P["w_head2"]), P["g_head2"], P["b_head2"], groups=1)
    return out[0], (d3, d2, d1)


def forward(hist, dt, P):
    """c(t + dt) = G([c(t-lb+1) .. c(t)])(dt)  (Eq. 1): hist [lb, H, W] -> [H, W]."""
    zc = condition(encode(hist, P), dt, P)
    return decode(zc, P)[0]


def forward_batch(hists, dts, P):
    return np.stack([forward(h, float(d), P) for h, d in zip(hists, dts)])
