"""GPU parity of the U-Net inference path (NEXT-4, include/unet.h) against the float64 oracle
(oracle/unet_oracle.py), through the C ABI.

Tolerances:
* one convolution (tcgen05 implicit GEMM, bf16 operands that are exactly representable, fp32
  accumulation over K = 9 cin <= 1152 products): normwise relative error <= 1e-5 (fp32 summation,
  ~sqrt(K) u_32 = 2e-6), every element within 1e-5 of the oracle's sum of |terms|;
* the whole network: activations are rounded to bf16 (u = 2^-9) at each of the 9 conv inputs and
  GroupNorm re-normalises every layer, so errors add up to ~9 u per layer chain: normwise
  relative error <= 2e-2 on the output (R-36).
Plus exact GPU-vs-GPU properties: batch members are independent (bitwise), the rollout equals the
composition of forward calls, w0 = 0 makes the output independent of dt."""
import numpy as np
import pytest

from paper_2312_05410_b200 import synth, unet
from oracle import unet_oracle as U

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    unet.lib()


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


@pytest.mark.parametrize("B,H,W,cin,cout", [(2, 24, 24, 16, 16), (1, 10, 13, 32, 32), (3, 16, 8, 48, 64),
                                            (1, 12, 12, 128, 128), (2, 9, 7, 256, 32), (1, 8, 16, 16, 128),
                                            # W % 128 == 0: the row-tile kernel (shifted descriptors)
                                            (1, 3, 128, 16, 16), (2, 2, 256, 32, 32), (1, 4, 128, 64, 16),
                                            (1, 5, 256, 16, 64), (2, 1, 128, 48, 128),
                                            # enough row tiles that every CTA's shared-memory ring
                                            # wraps (more iterations than stages)
                                            (8, 80, 128, 64, 16), (8, 160, 256, 16, 16),
                                            # rows of 32 / 64 pixels through the row kernel (one row
                                            # per 128-lane tile), cin up to 128
                                            (2, 20, 64, 128, 32), (3, 12, 32, 64, 128), (2, 16, 64, 32, 64),
                                            (9, 40, 64, 128, 16)])
def test_conv3x3_tensor_core_kernel(B, H, W, cin, cout):
    import torch
    g = np.random.default_rng(B * 1000 + cin + cout)
    x = synth.to_bf16(g.standard_normal((B, H, W, cin))).astype(np.float64)
    w = synth.to_bf16(g.standard_normal((cout, 3, 3, cin)) / np.sqrt(9 * cin)).astype(np.float64)
    dx = torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).cuda().contiguous()
    dw = torch.tensor(w, dtype=torch.float32).to(torch.bfloat16).cuda().contiguous()
    dout = torch.full((B, H, W, cout), float("nan"), dtype=torch.float32, device="cuda")
    unet.conv3x3(dx.data_ptr(), dw.data_ptr(), dout.data_ptr(), B, H, W, cin, cout)
    torch.cuda.synchronize()
    got = dout.cpu().numpy().astype(np.float64)
    for b in (range(B) if B < 8 else (0, B // 2 + 1, B - 1)):
        ref = U.conv(np.transpose(x[b], (2, 0, 1)), w)                       # [cout, H, W]
        mag = U.conv(np.abs(np.transpose(x[b], (2, 0, 1))), np.abs(w))
        gb = np.transpose(got[b], (2, 0, 1))
        assert np.all(np.isfinite(gb))
        assert _rel(gb, ref) <= 1e-5, (b, _rel(gb, ref))
        assert np.all(np.abs(gb - ref) <= 1e-5 * mag + 1e-30), b


def _net(H=32, W=32, batch=4, seed=21, lb=3, widths=(16, 32, 64, 128)):
    p = unet.default_params(height=H, width=W, max_batch=batch, lb=lb, widths=widths)
    blob = synth.random_weights(seed, lb, widths)
    return unet.UNet(p, blob), synth.unpack(blob, lb, widths)


@pytest.mark.parametrize("H,W,batch", [(32, 32, 3), (16, 40, 2)])
def test_forward_matches_oracle(H, W, batch):
    net, P = _net(H, W, batch)
    hist = synth.histories(batch, 3, H, W, seed=5)
    dts = np.array([1.0, 2.0, 3.0, 4.0][:batch])
    with net:
        got = net.forward(hist, dts)
        assert net.launches() > 0
    assert got.shape == (batch, H, W) and np.all(np.isfinite(got))
    for b in range(batch):
        ref = U.forward(hist[b], dts[b], P)
        assert _rel(got[b], ref) <= 2e-2, (b, _rel(got[b], ref))
        # elementwise: every output within 6e-2 of the output's scale (R-36: nine bf16 roundings
        # of re-normalised activations, u = 2^-9 each, ~1.8% worst case; x3 margin for the final
        # GroupNorm's division by a sample standard deviation)
        assert np.max(np.abs(got[b] - ref)) <= 6e-2 * np.max(np.abs(ref)), (b, np.max(np.abs(got[b] - ref)))


def test_forward_other_widths_and_lookback():
    widths = (16, 16, 32, 32)
    net, P = _net(24, 24, 2, seed=3, lb=5, widths=widths)
    hist = synth.histories(2, 5, 24, 24, seed=6)
    with net:
        got = net.forward(hist, np.array([0.5, 2.5]))
    for b, dt in enumerate((0.5, 2.5)):
        assert _rel(got[b], U.forward(hist[b], dt, P)) <= 2e-2


def test_host_forward_chunk_pipeline_equals_one_device_forward():
    """un_forward pipelines batches of >= 16 over 4 sample chunks (copies overlapped, one graph per
    chunk); the result equals one un_forward_device of the whole batch bitwise, also for a batch
    that does not split evenly, and with page-locked buffers."""
    import torch
    for B in (18, 20):
        net, _ = _net(32, 32, B, seed=23)
        hist = synth.histories(B, 3, 32, 32, seed=9).astype(np.float32)
        dts = (1.0 + np.arange(B) % 5).astype(np.float32)
        with net:
            host = net.forward(hist, dts)
            pinned = torch.empty((B, 32, 32), dtype=torch.float32).pin_memory().numpy()
            net.forward(torch.from_numpy(hist).pin_memory().numpy(), torch.from_numpy(dts).pin_memory().numpy(), pinned)
            dh, dd = torch.from_numpy(hist).cuda(), torch.from_numpy(dts).cuda()
            do = torch.empty((B, 32, 32), dtype=torch.float32, device="cuda")
            torch.cuda.synchronize()   # the ctx stream does not order against torch's stream
            net.forward_device(B, dh.data_ptr(), dd.data_ptr(), do.data_ptr())
            torch.cuda.synchronize()
            dev = do.cpu().numpy()
        assert np.array_equal(host, dev), B
        assert np.array_equal(pinned, dev), B


def test_batch_members_are_independent_and_deterministic():
    net, _ = _net(32, 32, 4)
    hist = synth.histories(4, 3, 32, 32, seed=8)
    dts = np.array([1.0, 3.0, 2.0, 5.0])
    with net:
        a = net.forward(hist, dts)
        b = net.forward(hist, dts)
        one = net.forward(hist[2:3], dts[2:3])
        perm = net.forward(hist[::-1].copy(), dts[::-1].copy())
    assert np.array_equal(a, b)
    assert np.array_equal(a[2], one[0])
    assert np.array_equal(a[::-1], perm)


def test_dt_constancy_when_w0_is_zero():
    P = synth.unpack(synth.random_weights(9))
    P["m_w0"] = np.zeros(128)
    p = unet.default_params(height=16, width=16, max_batch=2)
    hist = synth.histories(2, 3, 16, 16, seed=10)
    with unet.UNet(p, synth.pack(P)) as net:
        a = net.forward(hist, np.array([1.0, 1.0]))
        b = net.forward(hist, np.array([4.0, 7.0]))
    assert np.array_equal(a, b)


def test_rollout_is_composition_of_forward_calls():
    net, _ = _net(16, 16, 2)
    hist = synth.histories(2, 3, 16, 16, seed=11)
    lf, leaps = 4, 2
    with net:
        out = net.rollout(hist, lf, leaps)
        win = hist.astype(np.float32)
        for leap in range(leaps):
            preds = [net.forward(win, np.full(2, q + 1.0)) for q in range(lf)]
            for q in range(lf):
                assert np.array_equal(out[:, leap * lf + q], preds[q]), (leap, q)
            win = np.stack(preds[lf - 3:], axis=1)


def test_full_size_sampled_members():
    """configs of the bench: 256 x 256, batch 64; two members checked against the oracle."""
    p = unet.default_params()
    blob = synth.random_weights(1)
    P = synth.unpack(blob)
    hist = synth.histories(64, 3, 256, 256, seed=2)
    dts = 1.0 + np.arange(64) % 5
    with unet.UNet(p, blob) as net:
        got = net.forward(hist, dts)
    assert np.all(np.isfinite(got))
    for b in (0, 37):
        ref = U.forward(hist[b], dts[b], P)
        assert _rel(got[b], ref) <= 2e-2, b
        assert np.max(np.abs(got[b] - ref)) <= 6e-2 * np.max(np.abs(ref)), b


def test_hybrid_schedule_dns_then_surrogate():
    """un_hybrid: the DNS part equals pf_trajectory's composite snapshots, the surrogate part equals
    un_rollout from the last lb of them (bitwise), and both segments are timed."""
    from paper_2312_05410_b200 import pf
    p = pf.pf_default_params(2).replace(nx=32, ny=32, n_members=2, ic_height=10.0, check_every=50)
    n_dns, K, lf, leaps = 4, 5, 3, 2
    net, _ = _net(32, 32, 2)
    with net:
        with pf.Simulation(p) as s:
            out, (t_dns, t_sur) = net.hybrid(s, n_dns, K, lf, leaps)
            assert pf.pf_info(s.ctx)[0] == (n_dns - 1) * K
        with pf.Simulation(p) as s:
            ref = np.empty((2, n_dns, 32, 32))
            pf.pf_trajectory(s.ctx, n_dns, K, ref)
        assert np.array_equal(out[:, :n_dns], ref.astype(np.float32))
        roll = net.rollout(ref[:, n_dns - 3:].astype(np.float32), lf, leaps)
    assert np.array_equal(out[:, n_dns:], roll)
    assert out.shape == (2, n_dns + lf * leaps, 32, 32) and t_dns > 0 and t_sur > 0
