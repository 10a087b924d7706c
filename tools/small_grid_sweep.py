"""Cell-steps/s of the small-grid kernels -- band (kernel_path 6) and persistent tile (7) -- against the
pair kernel with CUDA graphs (kernel_path 3, graph_steps 50) over grid sizes: where the default
switches (kPersistentCells).  configs[0] (64^2, all mobilities 1) and configs[1] (256^2) are timed
with their own presets first."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rate(p, steps):
    import torch
    from paper_2312_05410_b200 import pf
    with pf.Simulation(p) as s:
        s.step(20)
        st = torch.cuda.ExternalStream(pf.pf_stream(s.ctx))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        s.step(steps)
        e1.record(st)
        torch.cuda.synchronize()
        return p.n_members * p.nx * p.ny * steps / (e0.elapsed_time(e1) * 1e-3)


def _try(p, steps):
    try:
        return rate(p, steps) / 1e9
    except Exception as e:   # the band kernel rejects grids whose bands do not fit
        return str(e)[:60]


def main():
    from paper_2312_05410_b200 import pf
    for cfg, steps in ((1, 1000), (2, 2000)):
        p = pf.pf_default_params(cfg)
        print(json.dumps({"config": cfg, "nx": p.nx, "steps": steps, "band_G": _try(p.replace(kernel_path=6), steps),
                          "persistent_G": _try(p.replace(kernel_path=7), steps),
                          "pair_graph_G": _try(p.replace(kernel_path=3, graph_steps=50), steps)}), flush=True)
    if "--only-configs" in sys.argv:   # configs[0] / configs[1] only (A/B runs)
        return
    for (n, m) in ((64, 1), (128, 1), (256, 1), (256, 4), (512, 1), (512, 4), (1024, 1)):
        p = pf.pf_default_params(2).replace(nx=n, ny=n, n_members=m, ic_height=n / 8, graph_steps=50, check_every=100)
        steps = 400 if n * n * m <= 1 << 18 else 200
        print(json.dumps({"nx": n, "members": m, "cells": n * n * m, "band_G": _try(p.replace(kernel_path=6), steps),
                          "persistent_G": _try(p.replace(kernel_path=7), steps),
                          "pair_graph_G": _try(p.replace(kernel_path=3), steps)}), flush=True)


if __name__ == "__main__":
    main()
