"""Small runs of each kernel path for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_case.py pair

cases: band (configs[0] 64^2, the band cluster kernel), persistent (64^2, cooperative tile kernel),
pair (512 x 72, 2 members: the TMA-ring stage kernels), loopback (512 x 72 in 2 y-slabs with the
overlap schedule), ws (warp-specialised step kernel), tile (fallback kernel), diag (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(case):
    import numpy as np
    from paper_2312_05410_b200 import pf
    small = pf.pf_default_params(2).replace(nx=512, ny=72, ic_height=18.0, n_members=2, graph_steps=0,
                                            check_every=3, rate_lo=0.5, rate_hi=2.0)
    if case == "band":
        p, mode, n = pf.pf_default_params(1).replace(kernel_path=6, check_every=3), "single", 4
    elif case == "persistent":
        p, mode, n = pf.pf_default_params(1).replace(kernel_path=7, check_every=3), "single", 4
    elif case == "pair":
        p, mode, n = small.replace(kernel_path=3), "single", 3
    elif case == "loopback":
        p, mode, n = small.replace(kernel_path=3, overlap_halo=1, ny=64), ("loopback", 2), 3
    elif case == "ws":
        p, mode, n = small.replace(kernel_path=5), "single", 3
    elif case == "tile":
        p, mode, n = small.replace(kernel_path=1), "single", 3
    else:
        raise SystemExit(f"unknown case {case}")
    with pf.Simulation(p, mode) as s:
        s.step(n)
        u = s.fields(0)
        d = s.diagnostics(0)
    assert all(np.all(np.isfinite(f)) for f in u) and d[4] == 0
    print(f"{case}: ok ({n} steps)")


if __name__ == "__main__":
    main(sys.argv[1])
