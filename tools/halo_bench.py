"""Halo-exchange cost on one GPU: configs[3] (4096^2 fp64) split into P loopback y-slabs, per-step
time with the device-copy transport (halo_transport 0) and the B11 peer-store transport
(halo_transport 1, push kernel + arrival counters + cuStreamWaitValue32), with and without the
overlap schedule.  The slabs of a loopback ctx share one GPU, so the compute per step is the same
for every P; ms_per_step(P) - ms_per_step(1) is what the decomposition and its exchange add.

    python tools/halo_bench.py [--steps 100] [--slabs 1,2,4,8] > halo.jsonl

pf_step is synchronous; each line is the median of 3 wall-clock timed pf_step(steps) calls
after one untimed call (the host enqueues every launch of a call up front, so the time is the
device's)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2312_05410_b200 import pf
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--slabs", default="1,2,4,8")
    args = ap.parse_args()
    base = pf.pf_default_params(args.config).replace(graph_steps=0, check_every=1000000)
    cells = base.nx * base.ny * base.n_members
    for P in [int(x) for x in args.slabs.split(",")]:
        for transport in ((0,) if P == 1 else (0, 1, 2)):
            for overlap in ((1,) if P == 1 else (1, 0)):
                p = base.replace(halo_transport=transport, overlap_halo=overlap)
                mode = "single" if P == 1 else ("loopback", P)
                with pf.Simulation(p, mode) as s:
                    s.step(args.steps)
                    runs = []
                    for _ in range(3):
                        t0 = time.perf_counter()
                        s.step(args.steps)
                        runs.append((time.perf_counter() - t0) * 1e3)
                    launches = pf.pf_launch_count(s.ctx)
                ms = sorted(runs)[1] / args.steps
                print(json.dumps({"config": args.config, "nx": p.nx, "ny": p.ny, "slabs": P,
                                  "halo_transport": transport, "overlap": overlap, "ms_per_step": ms,
                                  "cell_updates_per_s": cells / ms * 1e3, "runs_ms": runs,
                                  "launches_total": launches}), flush=True)


if __name__ == "__main__":
    main()
