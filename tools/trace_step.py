"""Phase timeline of the small-grid step kernel (kernel_path 7; diagnostic build with -DPF_TRACE=1,
loaded through PF_LIB): per phase the median over blocks and steps of its duration (ns), and the
grid-barrier wait split into the block's own idle time and the barrier's latency.

    PF_LIB=.../libpf_trace.so python tools/trace_step.py [config] [nx]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PHASES = ["load", "a2_stage1", "ustar", "a2_stage2", "stage2_store"]


def main():
    import numpy as np
    from paper_2312_05410_b200 import pf
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    p = pf.pf_default_params(cfg).replace(kernel_path=7, check_every=1000, graph_steps=0)
    if len(sys.argv) > 2:
        n = int(sys.argv[2])
        p = p.replace(nx=n, ny=n, ic_height=n / 8)
    with pf.Simulation(p) as s:
        s.step(64)
        s.step(64)
        buf = np.zeros((160, 64, 8), dtype=np.int64)
        rc = pf.lib().pf_debug_step_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong)))
    assert rc == 0, rc
    used = buf[:, 8:, 0] > 0
    nb = int(used[:, 0].sum())
    b = buf[:nb, 8:, :]
    out = {"config": cfg, "nx": p.nx, "blocks_traced": nb}
    for k, name in enumerate(PHASES):
        out[name + "_ns"] = float(np.median(b[:, :, k + 1] - b[:, :, k]))
    # grid barrier: from a block's tile end to its own release, and the latest tile end of the step
    # to the earliest release (the barrier's own latency)
    out["barrier_wait_ns"] = float(np.median(b[:, :, 6] - b[:, :, 5]))
    last_end = b[:, :, 5].max(axis=0)
    first_rel = b[:, :, 6].min(axis=0)
    out["barrier_latency_ns"] = float(np.median(first_rel - last_end))
    out["tile_end_spread_ns"] = float(np.median(last_end - b[:, :, 5].min(axis=0)))
    step = b[:, 1:, 6].min(axis=0) - b[:, :-1, 6].min(axis=0)
    out["step_ns"] = float(np.median(step))
    out["start_after_release_ns"] = float(np.median(b[:, 1:, 0] - b[:, :-1, 6]))
    out["loop_top_after_release_ns"] = float(np.median(b[:, 1:, 7] - b[:, :-1, 6]))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
