import sys, time, json
sys.path.insert(0, '.')
import torch
from paper_2312_05410_b200 import pf
p = pf.pf_default_params(3)
for graph in (0, 25):
    for prof in (False, True):
        q = p.replace(graph_steps=graph)
        with pf.Simulation(q) as s:
            s.step(20)
            stream = torch.cuda.ExternalStream(pf.pf_stream(s.ctx))
            if prof: pf.pf_profile(s.ctx, True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream); s.step(200); e1.record(stream); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            st = pf.pf_profile_read(s.ctx) if prof else None
            print(json.dumps({"graph": graph, "prof": prof, "ms_per_step": ms / 200,
                              "stage_sum_per_step": (st[0] + st[2]) / 200 if prof else None}))
