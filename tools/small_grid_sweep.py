"""Cell-steps/s of the persistent small-grid kernel (kernel_path 7) against the pair kernel with CUDA
graphs (kernel_path 3, graph_steps 50) over grid sizes: where the default switches (kPersistentCells)."""
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


def main():
    from paper_2312_05410_b200 import pf
    for (n, m) in ((64, 1), (128, 1), (256, 1), (256, 4), (512, 1), (512, 4), (1024, 1)):
        p = pf.pf_default_params(2).replace(nx=n, ny=n, n_members=m, ic_height=n / 8, graph_steps=50, check_every=100)
        steps = 400 if n * n * m <= 1 << 18 else 200
        a = rate(p.replace(kernel_path=7), steps)
        b = rate(p.replace(kernel_path=3), steps)
        print(json.dumps({"nx": n, "members": m, "cells": n * n * m, "persistent_G": a / 1e9, "pair_graph_G": b / 1e9}),
              flush=True)


if __name__ == "__main__":
    main()
