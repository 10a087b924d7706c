"""Seeded synthetic inputs for the temporally conditioned U-Net.

No arithmetic of the method lives here: only the parameter list of the network (names, shapes,
order of the flat weight blob), seeded random draws rounded to bfloat16-representable values, and
synthetic look-back histories.  Both the oracle tests and the GPU path receive the same arrays;
trained weights do not exist (P:470-483 trains on a dataset that is absent), so every weight is
random.

Network (readings R-29..R-36): look-back lb channels, level widths C1..C4, a 128-wide
time-basis MLP, conv 3x3 'same' convolutions without bias, GroupNorm with G groups, 2x2 up-sampling
with one 2x2 kernel per up operation.
"""
from __future__ import annotations

import numpy as np

BASIS = 128          # width of the time-basis MLP ("2 hidden layers with 128 neurons")


def arch(lb=3, widths=(16, 32, 64, 128)):
    """Layer table [(name, cin, cout)] of the conv layers, in execution order."""
    c1, c2, c3, c4 = widths
    return [("enc1", lb, c1), ("enc2", c1, c2), ("enc3", c2, c3), ("enc4", c3, c4),
            ("dec4", c4, c3), ("dec3", 2 * c3, c2), ("dec2", 2 * c2, c1), ("head1", 2 * c1, c1),
            ("head2", c1, 1)]


def param_shapes(lb=3, widths=(16, 32, 64, 128)):
    """Ordered (name, shape) list of the flat float32 weight blob.

    conv weights  w_<layer>  [cout, 3, 3, cin]   (K index = (ky*3 + kx)*cin + ci)
    GroupNorm     g_<layer>, b_<layer> [cout]     (gamma, beta)
    projections   wl1..wl4   [C_p, 128]           (w^{L_p}, no bias)
    up kernels    up3, up2, up1 [2, 2]            (w^{tconv} of d^{L3}, d^{L2}, d^{L1})
    time MLP      m_w0 [128], m_b0 [128], m_w1 [128,128], m_b1 [128], m_w2 [128,128], m_b2 [128]
    """
    out = []
    for name, ci, co in arch(lb, widths):
        out += [("w_" + name, (co, 3, 3, ci)), ("g_" + name, (co,)), ("b_" + name, (co,))]
    for p, c in enumerate(widths, 1):
        out.append((f"wl{p}", (c, BASIS)))
    out += [("up3", (2, 2)), ("up2", (2, 2)), ("up1", (2, 2))]
    out += [("m_w0", (BASIS,)), ("m_b0", (BASIS,)), ("m_w1", (BASIS, BASIS)), ("m_b1", (BASIS,)),
            ("m_w2", (BASIS, BASIS)), ("m_b2", (BASIS,))]
    return out


def blob_size(lb=3, widths=(16, 32, 64, 128)):
    return int(sum(np.prod(s) for _, s in param_shapes(lb, widths)))


def to_bf16(a):
    """Round float values to the nearest bfloat16 (ties to even), returned as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def random_weights(seed, lb=3, widths=(16, 32, 64, 128)):
    """Flat float32 blob of bf16-representable random weights (fan-in scaled normal draws)."""
    g = np.random.default_rng(seed)
    parts = []
    for name, shape in param_shapes(lb, widths):
        n = int(np.prod(shape))
        if name.startswith("w_"):
            fan = shape[1] * shape[2] * shape[3]
            v = g.standard_normal(n) * np.sqrt(2.0 / fan)
        elif name.startswith("g_"):
            v = 1.0 + 0.1 * g.standard_normal(n)
        elif name.startswith("b_"):
            v = 0.1 * g.standard_normal(n)
        elif name.startswith("wl"):
            v = g.standard_normal(n) / np.sqrt(BASIS)
        elif name.startswith("up"):
            v = 0.5 + 0.25 * g.standard_normal(n)
        elif name == "m_w0":
            v = 2.0 * g.standard_normal(n)
        elif name in ("m_w1", "m_w2"):
            v = g.standard_normal(n) / np.sqrt(BASIS)
        else:
            v = 0.5 * g.standard_normal(n)
        parts.append(v)
    return to_bf16(np.concatenate(parts))


def unpack(blob, lb=3, widths=(16, 32, 64, 128)):
    """Dict name -> float64 array view of the blob (shapes of param_shapes)."""
    blob = np.asarray(blob, dtype=np.float64)
    out, o = {}, 0
    for name, shape in param_shapes(lb, widths):
        n = int(np.prod(shape))
        out[name] = blob[o:o + n].reshape(shape)
        o += n
    assert o == blob.size, (o, blob.size)
    return out


def pack(params, lb=3, widths=(16, 32, 64, 128)):
    """Inverse of unpack (float32 blob)."""
    return np.concatenate([np.asarray(params[n], dtype=np.float32).ravel()
                           for n, _ in param_shapes(lb, widths)])


def histories(batch, lb, h, w, seed):
    """[batch, lb, h, w] look-back windows of composite-c-like fields in [0, 1] (bf16-representable):
    a smooth film with a random rough top, c = 0 above it (vapour), c in (0.2, 0.8) inside."""
    g = np.random.default_rng(seed)
    y = np.arange(h)[:, None] * np.ones((1, w))
    x = np.arange(w)[None, :] * np.ones((h, 1))
    out = np.zeros((batch, lb, h, w))
    for b in range(batch):
        H0 = h * (0.3 + 0.3 * g.random())
        ph = g.random(4) * 2 * np.pi
        for t in range(lb):
            top = H0 + t * 0.5 + 0.05 * h * (np.sin(2 * np.pi * x / w + ph[0]) + 0.5 * np.sin(6 * np.pi * x / w + ph[1]))
            solid = y < top
            c = 0.5 + 0.3 * np.sin(2 * np.pi * 3 * x / w + ph[2]) * np.cos(2 * np.pi * y / h + ph[3])
            c = c + 0.02 * g.standard_normal((h, w))
            out[b, t] = np.where(solid, np.clip(c, 0.0, 1.0), 0.0)
    return to_bf16(out).astype(np.float64)
