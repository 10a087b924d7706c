"""NEXT-1 measurement: dataset-generation throughput of pf_trajectory on the paper's workload shape
(256^2 mesh, per-member deposition rate v in [0.3, 1.0], angle in [50, 90] degrees and
species mobilities (R-23: M_A, M_B scaled by [0.5, 1]),
50 equally spaced snapshots of the composite field), against plain stepping of the same ensemble.

    python tools/dataset_bench.py [--members 64] [--snapshots 50] [--every 20]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2312_05410_b200 import pf
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=64)
    ap.add_argument("--snapshots", type=int, default=50)
    ap.add_argument("--every", type=int, default=20)
    a = ap.parse_args()
    p = pf.pf_default_params(2).replace(n_members=a.members, v0=0.5, rate_lo=0.6, rate_hi=2.0, theta_deg=50.0,
                                       theta_span=40.0, mob_lo=0.5, mob_hi=1.0, seed=2024)
    cells = p.n_members * p.nx * p.ny
    steps = (a.snapshots - 1) * a.every
    out = torch.empty((p.n_members, a.snapshots, p.ny, p.nx), dtype=torch.float64).pin_memory()
    res = {"members": p.n_members, "grid": [p.ny, p.nx], "snapshots": a.snapshots, "steps_between": a.every,
           "steps": steps, "snapshot_bytes": out.numel() * 8}
    with pf.Simulation(p) as s:
        s.step(5)
        stream = torch.cuda.ExternalStream(pf.pf_stream(s.ctx))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        s.step(steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_plain = e0.elapsed_time(e1)
        t0 = time.perf_counter()
        pf.pf_trajectory(s.ctx, a.snapshots, a.every, out)
        ms_traj = 1e3 * (time.perf_counter() - t0)
        # the same trajectory streamed to a file (float32, the dataset's storage), writer thread
        # overlapping the stepping
        import tempfile
        path = os.path.join(tempfile.mkdtemp(), "dataset.pftraj")
        t0 = time.perf_counter()
        pf.pf_trajectory_file(s.ctx, path, a.snapshots, a.every, "float32")
        ms_file = 1e3 * (time.perf_counter() - t0)
        file_bytes = os.path.getsize(path)
        os.remove(path)
    res.update({"ms_trajectory_file_f32": ms_file, "file_bytes": file_bytes,
                "trajectories_per_s_file": p.n_members / (ms_file * 1e-3)})
    res.update({"ms_plain": ms_plain, "ms_trajectory": ms_traj,
                "cell_updates_per_s_plain": cells * steps / (ms_plain * 1e-3),
                "cell_updates_per_s_trajectory": cells * steps / (ms_traj * 1e-3),
                "trajectories_per_s": p.n_members / (ms_traj * 1e-3),
                "snapshot_overhead": ms_traj / ms_plain - 1.0})
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
