"""Measurement of the NEXT-4 row: temporally conditioned U-Net inference (include/unet.h).

    python tools/unet_bench.py [--batch 64] [--hw 256] [--iters 20] [--warmup 3] [--no-cpu]

Workload: the paper's grid (256 x 256), look-back lb = 3, widths (16, 32, 64, 128), random
bf16 weights (no trained weights exist), a batch of seeded synthetic histories with dt = 1..5.
Prints one JSON line: samples/s with inputs resident on the device (CUDA events on the ctx
stream), the roofline of the convolution kernels (algorithmic bytes / their event time against
the measured HBM bandwidth; the tensor-core FLOP rate is reported beside it), the end-to-end rate through un_forward with host buffers,
the oracle's single-thread rate on one sample (cpu_baseline) and the sampled parity error.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--hw", type=int, default=256)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch
    from bench import ClockSampler
    from paper_2312_05410_b200 import synth, unet

    B, HW = a.batch, a.hw
    p = unet.default_params(height=HW, width=HW, max_batch=B)
    blob = synth.random_weights(1)
    hist = synth.histories(B, 3, HW, HW, seed=2).astype(np.float32)
    dts = (1.0 + np.arange(B) % 5).astype(np.float32)
    net = unet.UNet(p, blob)
    st = torch.cuda.ExternalStream(net.stream())
    dh = torch.from_numpy(hist).cuda()
    dd = torch.from_numpy(dts).cuda()
    do = torch.empty((B, HW, HW), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    for _ in range(a.warmup):
        net.forward_device(B, dh.data_ptr(), dd.data_ptr(), do.data_ptr())
    torch.cuda.synchronize()
    l0 = net.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(st)
        for _ in range(a.iters):
            net.forward_device(B, dh.data_ptr(), dd.data_ptr(), do.data_ptr())
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    launches = (net.launches() - l0) / a.iters
    # profiled pass: conv kernels' share (events around every conv launch)
    net.profile(True)
    for _ in range(5):
        net.forward_device(B, dh.data_ptr(), dd.data_ptr(), do.data_ptr())
    conv_ms, fwd_ms, nf, flops = net.profile_read()
    net.profile(False)
    conv_ms, fwd_ms = conv_ms / nf, fwd_ms / nf
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak_tf, peak_bw = float(peaks["bf16_tflops"]), float(peaks["hbm_gbs"])
    tflops = flops * B / (conv_ms * 1e-3) / 1e12
    # algorithmic bytes of the 9 convolutions per sample: bf16 input activations read once, fp32
    # output written once; the arithmetic intensity (<= 48 flop/B at 16 channels)
    # is far below the B200 balance point, so the convolutions are HBM-bound
    c1, c2, c3, c4 = 16, 32, 64, 128
    layers = [(3, c1, 0), (c1, c2, 1), (c2, c3, 2), (c3, c4, 3), (c4, c3, 3), (2 * c3, c2, 2), (2 * c2, c1, 1),
              (2 * c1, c1, 0), (c1, 1, 0)]
    conv_bytes = sum((HW >> lv) * (HW >> lv) * (2 * ci + 4 * co) for ci, co, lv in layers)
    achieved = conv_bytes * B / (conv_ms * 1e-3) / 1e9
    # end to end: page-locked host buffers through un_forward (H2D of the histories and dt, D2H of
    # the predictions, pipelined over sample chunks inside the call)
    hist_p = torch.from_numpy(hist).pin_memory().numpy()
    dts_p = torch.from_numpy(dts).pin_memory().numpy()
    out_p = torch.empty((B, HW, HW), dtype=torch.float32).pin_memory().numpy()
    net.forward(hist_p, dts_p, out_p)
    t0 = time.perf_counter()
    n_e2e = max(3, a.iters // 4)
    for _ in range(n_e2e):
        net.forward(hist_p, dts_p, out_p)
    e2e = B * n_e2e / (time.perf_counter() - t0)
    out = out_p
    # sampled parity
    from oracle import unet_oracle as U
    P = synth.unpack(blob)
    errs = []
    for b in (0, B - 1):
        ref = U.forward(hist[b].astype(np.float64), float(dts[b]), P)
        errs.append(float(np.linalg.norm(out[b] - ref) / np.linalg.norm(ref)))
    res = {
        "metric": "U-Net (temporal conditioning) inference samples/s, 256x256, lb=3, batch 64",
        "value": B / (ms * 1e-3), "unit": "samples/s", "ms_per_forward": ms, "batch": B,
        "higher_is_better": True, "dtype": "bf16 (fp32 accumulate, GN statistics fp64 across 32-pixel units)", "data": "synthetic",
        "config": {"workload": f"U-Net TC forward, {B} x {HW}x{HW}, lb=3, widths 16/32/64/128, random bf16 weights",
                   "l2": "activations > 126 MB L2 at batch 64"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_bw, "unit": "GB/s",
                     "frac": achieved / peak_bw, "traffic": None,
                     "kernel": "conv3x3 kernels (all 9 convolutions of a forward)", "conv_ms": conv_ms,
                     "forward_ms_profiled": fwd_ms, "conv_share": conv_ms / fwd_ms,
                     "bytes_per_sample": conv_bytes, "flops_per_sample": flops,
                     "tensor_tflops": tflops, "tensor_frac": tflops / peak_tf},
        "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": hist.nbytes + dts.nbytes,
                "d2h_bytes_per_step": B * HW * HW * 4,
                "note": "un_forward with page-locked host buffers (histories, dt, predictions); copies "
                        "pipelined against the forward over 4 sample chunks inside the call; wall clock "
                        "over the calls"},
        "gpu_launches": launches,
        "parity_rel_l2": errs,
        "clocks": clk.summary(),
    }
    if not a.no_cpu:
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < 10.0 or n == 0:
            U.forward(hist[n % B].astype(np.float64), float(dts[n % B]), P)
            n += 1
        el = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": n / el, "unit": "samples/s", "cores": 1, "kind": "oracle",
                               "sample": f"{n} samples of the workload, numpy float64 oracle, {el:.1f} s"}
    net.close()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
