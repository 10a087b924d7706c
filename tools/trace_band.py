"""Phase timeline of the band kernel (kernel_path 6) on configs[0] (diagnostic build with
-DPF_TRACE=1 through PF_LIB): median cycles per stage of phase A (mu/M), phase B (update), phase C
(stores + DSMEM pushes + cluster barrier) and the stage total, over 16 blocks x 120 stages.
    PF_LIB=.../libpf_trace.so python tools/trace_band.py"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    from paper_2312_05410_b200 import pf
    p = pf.pf_default_params(1).replace(kernel_path=6, check_every=1000, graph_steps=0)
    with pf.Simulation(p) as s:
        s.step(64)
        s.step(64)
        buf = np.zeros((16, 128, 4), dtype=np.int64)
        assert pf.lib().pf_debug_band_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
    b = buf[:, 8:, :]
    a = b[:, :, 0] - b[:, :, 3]
    bb = b[:, :, 1] - b[:, :, 0]
    cc = b[:, :, 2] - b[:, :, 1]
    tot = b[:, 1:, 3] - b[:, :-1, 3]
    wait = b[:, 1:, 3] - b[:, :-1, 2]   # P2P builds: the halo wait (stage end to next stage start)
    print(json.dumps({"phase_A_cyc": float(np.median(a)), "phase_B_cyc": float(np.median(bb)),
                      "phase_C_cyc": float(np.median(cc)), "stage_cyc": float(np.median(tot)),
                      "phase_C_max_over_blocks_cyc": float(np.median(cc.max(axis=0))),
                      "halo_wait_cyc": float(np.median(wait))}))


if __name__ == "__main__":
    main()
