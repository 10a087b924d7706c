"""Timeline of one block of the fp64 stage-1 pair kernel (diagnostic build with -DPF_TRACE=1, loaded
through PF_LIB): producer wait / TMA issue times and the compute warps' full-barrier waits per box.

    PF_LIB=.../libpf_trace.so python tools/trace_stage1.py [config]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    from paper_2312_05410_b200 import pf
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    p = pf.pf_default_params(cfg).replace(check_every=1000, graph_steps=0)
    with pf.Simulation(p) as s:
        s.step(3)
        buf = np.zeros((5, 512, 2), dtype=np.int64)
        rc = pf.lib().pf_debug_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong)))
    assert rc == 0, rc
    sp = np.zeros((1024, 3), dtype=np.int64)
    assert pf.lib().pf_debug_block_spans(sp.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
    t0 = buf[buf > 0].min()
    tr = np.where(buf > 0, buf - t0, -1)
    nb = int((tr[4, :, 1] >= 0).sum())
    out = {"boxes": nb, "producer_issue_ns": tr[4, :nb, 1].tolist(), "producer_wait_ns": tr[4, :nb, 0].tolist()}
    for w in range(4):
        n = int((tr[w, :, 1] >= 0).sum())
        if n == 0:
            continue
        ws, we = tr[w, :n, 0], tr[w, :n, 1]
        waited = we - ws
        out[f"warp{w}"] = {"boxes": n, "wait_ns_total": int(waited.sum()), "span_ns": int(we[-1] - ws[0]),
                           "wait_start": ws.tolist(), "wait_end": we.tolist()}
        # latency from TMA issue to the end of the consumer's wait, for boxes the warp waited on
        lat = [int(we[g] - tr[4, g, 1]) for g in range(min(n, nb)) if waited[g] > 200]
        out[f"warp{w}"]["issue_to_ready_ns_when_waiting"] = lat[:64]
    nblk = int((sp[:, 0] > 0).sum())
    sp = sp[:nblk]
    t00 = sp[:, 0].min()
    out["blocks"] = nblk
    out["block_start_ns"] = [int(v) for v in np.percentile(sp[:, 0] - t00, [0, 10, 50, 90, 100])]
    out["block_end_ns"] = [int(v) for v in np.percentile(sp[:, 2] - t00, [0, 10, 50, 90, 100])]
    out["block_span_ns"] = [int(v) for v in np.percentile(sp[:, 2] - sp[:, 0], [0, 10, 50, 90, 100])]
    out["spans"] = (sp[:, 2] - sp[:, 0]).tolist()
    out["smid"] = sp[:, 1].tolist()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
