"""e2e (pf_run_host) timing vs member-chunk count on configs[2]."""
import sys, json
sys.path.insert(0, '.')
import torch
from paper_2312_05410_b200 import pf
p = pf.pf_default_params(3)
with pf.Simulation(p) as s:
    s.step(10)
    stream = torch.cuda.ExternalStream(pf.pf_stream(s.ctx))
    shp = (p.n_members, p.ny, p.nx)
    hin = [torch.empty(shp, dtype=torch.float64).pin_memory() for _ in range(3)]
    hout = [torch.empty(shp, dtype=torch.float64).pin_memory() for _ in range(3)]
    pf.pf_get_fields(s.ctx, -1, *hin)
    for chunks in (1, 2, 3, 4, 8):
        pf.pf_run_host(s.ctx, 5, *hin, *hout, chunks)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pf.pf_run_host(s.ctx, 200, *hin, *hout, chunks)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"chunks": chunks, "ms": ms, "e2e_G": 64 * 512 * 512 * 200 / ms / 1e6}))
