"""NEXT-2 measurement: S2 autocorrelation maps + radial profiles of dataset snapshots (256^2 composite
fields, the paper's mesh) on the GPU (pf_s2: cuFFT + own kernels, host buffers in and out) against the
oracle (numpy FFT, one thread) on a sample.  python tools/stats_bench.py [--fields 1024]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2312_05410_b200 import pf
    from oracle import oracle as ora
    ap = argparse.ArgumentParser()
    ap.add_argument("--fields", type=int, default=1024)
    a = ap.parse_args()
    p = pf.pf_default_params(2).replace(n_members=a.fields // 8, rate_lo=0.6, rate_hi=2.0, theta_deg=50.0,
                                       theta_span=40.0, seed=7)
    with pf.Simulation(p) as s:
        out = np.empty((p.n_members, 8, p.ny, p.nx))
        pf.pf_trajectory(s.ctx, 8, 200, out)
    comp = out.reshape(-1, p.ny, p.nx)
    pf.pf_s2(comp[:8])
    t0 = time.perf_counter()
    s2, rad = pf.pf_s2(comp)
    gpu_s = time.perf_counter() - t0
    k = 16
    t0 = time.perf_counter()
    for b in range(k):
        ora.radial_average(ora.s2_fft(ora.indicator(comp[b])))
    ora_s = time.perf_counter() - t0
    print(json.dumps({"fields": comp.shape[0], "grid": [p.ny, p.nx], "gpu_s": gpu_s,
                      "gpu_fields_per_s": comp.shape[0] / gpu_s, "oracle_sample": k,
                      "oracle_fields_per_s": k / ora_s, "note": "GPU time includes H2D of the fields and D2H of maps and profiles"}))


if __name__ == "__main__":
    main()
