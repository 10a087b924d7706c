"""Wall time of the paper's hybrid configurations on one B200 (section 2.4): DNS alone for
all snapshots vs DNS for the first n_dns snapshots and the U-Net (random weights: throughput
only) for the rest.

    python tools/hybrid_bench.py [--members 64] [--n 256] [--snapshots 50] [--steps-between 200]

The DNS is configs[1]'s model (256 x 256 fp64, M_c/M_phi = 10) with `members` ensemble members
(one trajectory each, the dataset layout of P:352-355); the surrogate rolls out from the last
lb = 3 DNS snapshots with lf = snapshots - n_dns forecasts in one leap.  Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=64)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--snapshots", type=int, default=50)
    ap.add_argument("--steps-between", type=int, default=200)
    a = ap.parse_args()
    import time
    import numpy as np
    from paper_2312_05410_b200 import pf, synth, unet
    p = pf.pf_default_params(2).replace(nx=a.n, ny=a.n, n_members=a.members, ic_height=a.n / 8,
                                        theta_span=40.0, theta_deg=50.0, rate_lo=0.3, rate_hi=1.0)
    S, K = a.snapshots, a.steps_between
    res = {"workload": f"{a.members} x {a.n}^2 fp64 DNS trajectories, {S} snapshots, {K} steps apart; "
                       f"U-Net lb=3, random bf16 weights", "members": a.members}
    with pf.Simulation(p) as s:
        s.step(10)                       # warm-up (graph / kernel set-up)
        out = np.empty((a.members, S, a.n, a.n))
        t0 = time.perf_counter()
        pf.pf_trajectory(s.ctx, S, K, out)
        res["dns_only_s"] = time.perf_counter() - t0
    net = unet.UNet(unet.default_params(height=a.n, width=a.n, max_batch=a.members), synth.random_weights(1))
    with net:
        for n_dns in (3, 10):            # the two configurations of P:240-241
            with pf.Simulation(p) as s:
                s.step(10)
                net.hybrid(s, 3, 1, S - n_dns, 1)             # warm-up of both paths (same shapes)
                _, (td, tu) = net.hybrid(s, n_dns, K, S - n_dns, 1)
            res[f"hybrid_dns{n_dns}"] = {"dns_s": td, "surrogate_s": tu, "speedup": res["dns_only_s"] / (td + tu)}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
