"""configs[3] as P loopback y-slabs on one GPU: per-step time of the NCCL send-to-self transport
(halo_transport 2) against the device-copy transport (0), direct launches and CUDA graphs
(PF_NCCL_SELF_GRAPH=1 lets transport 2 capture its NCCL groups), several repeats to show the spread.

    PF_NCCL_SELF_GRAPH=1 python tools/nccl_self_bench.py [--slabs 2] [--steps 200] > out.jsonl"""
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
    ap.add_argument("--slabs", type=int, default=2)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--reps", type=int, default=6)
    args = ap.parse_args()
    base = pf.pf_default_params(4).replace(check_every=1000000, overlap_halo=1)
    for transport in (0, 2):
        for graph in (0, 8):
            p = base.replace(halo_transport=transport, graph_steps=graph)
            with pf.Simulation(p, ("loopback", args.slabs)) as s:
                s.step(40)
                runs = []
                for _ in range(args.reps):
                    t0 = time.perf_counter()
                    s.step(args.steps)
                    runs.append((time.perf_counter() - t0) * 1e3 / args.steps)
            print(json.dumps({"slabs": args.slabs, "halo_transport": transport, "graph_steps": graph,
                              "self_graph_env": os.environ.get("PF_NCCL_SELF_GRAPH", "0"),
                              "ms_per_step_runs": [round(r, 4) for r in runs]}), flush=True)


if __name__ == "__main__":
    main()
