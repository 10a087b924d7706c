"""Kernel microbenchmark: per-stage CUDA-event times of the stage kernels on a preset.

    python tools/kbench.py [--config 3] [--path 0|1|2] [--steps 50] [--sweep]

--sweep re-runs itself in subprocesses over PF_STREAM_W / PF_STREAM_S settings."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(args):
    from paper_2312_05410_b200 import pf
    p = pf.pf_default_params(args.config).replace(kernel_path=args.path, graph_steps=0,
                                                  check_every=1000000)
    if args.members:
        p = p.replace(n_members=args.members)
    if args.nx:
        p = p.replace(nx=args.nx, ny=args.ny or args.nx)
    with pf.Simulation(p) as s:
        s.step(5)
        pf.pf_profile(s.ctx, True)
        s.step(args.steps)
        pr = pf.pf_profile_read(s.ctx)
    cells = p.n_members * p.nx * p.ny
    esz = 8 if p.precision == 0 else 4
    ms1, ms2 = pr[0] / pr[1], pr[2] / pr[3]
    out = {"cfg": args.config, "nx": p.nx, "ny": p.ny, "members": p.n_members,
           "path": args.path, "ms_stage1": ms1, "ms_stage2": ms2,
           "GBs_stage1": cells * 6 * esz / ms1 / 1e6, "GBs_stage2": cells * 9 * esz / ms2 / 1e6,
           "Gcell_steps_per_s": cells / (ms1 + ms2) / 1e6}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--path", type=int, default=0)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--members", type=int, default=0)
    ap.add_argument("--nx", type=int, default=0)
    ap.add_argument("--ny", type=int, default=0)
    ap.add_argument("--sweep", action="store_true")
    args = ap.parse_args()
    if not args.sweep:
        return one(args)
    combos = [{"PF_STREAM_S1": "12", "PF_STREAM_S2": "8"}, {"PF_STREAM_S1": "6", "PF_STREAM_S2": "6"},
              {"PF_STREAM_S1": "9", "PF_STREAM_S2": "7"}, {"PF_STREAM_S1": "15", "PF_STREAM_S2": "8"}]
    for c in combos:
        env = dict(os.environ)
        env.update(c)
        cmd = [sys.executable, __file__, "--config", str(args.config), "--steps", str(args.steps), "--path", "2"]
        if args.members:
            cmd += ["--members", str(args.members)]
        print(json.dumps(c), flush=True)
        subprocess.run(cmd, env=env)


if __name__ == "__main__":
    main()
