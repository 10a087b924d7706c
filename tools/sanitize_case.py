"""Small runs of each kernel path, for the checked build (PF_LIB=paper_2312_05410_b200/_variants/
libpf_checked.so: device bounds checks that trap + guard zones around the state buffers, checked
here through pf_debug_guards) or for compute-sanitizer where a pool allows it:

    PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_checked.so python tools/sanitize_case.py pair

cases: band (configs[0] 64^2, the band cluster kernel), persistent (64^2, cooperative tile kernel),
pair (512 x 72, 2 members: the TMA-ring stage kernels), loopback (512 x 72 in 2 y-slabs with the
overlap schedule; peer / nccl_self: the same with halo transport 1 / 2), ws (warp-specialised step kernel), tile (fallback kernel), diag (diagnostics)."""
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
    elif case == "peer":       # loopback slabs, B11 peer-store transport
        p, mode, n = small.replace(kernel_path=3, overlap_halo=1, ny=64, halo_transport=1), ("loopback", 2), 3
    elif case == "nccl_self":  # loopback slabs exchanging through NCCL sends to self (transport 2)
        p, mode, n = small.replace(kernel_path=3, overlap_halo=1, ny=64, halo_transport=2), ("loopback", 2), 3
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
        guard, bad = pf.pf_debug_guards(s.ctx)
    assert all(np.all(np.isfinite(f)) for f in u) and d[4] == 0
    assert bad == 0, f"{bad} guard bytes overwritten"
    print(f"{case}: ok ({n} steps, guard zones of {guard} B intact)")


if __name__ == "__main__":
    main(sys.argv[1])
