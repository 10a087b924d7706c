"""Two-rank NCCL slab decomposition on real GPUs (BASELINE configs[3]): one process per
GPU, pf_create_slab with an NCCL communicator, the 2-row halo exchanged per stage over NCCL and
overlapped with the interior update.  The gathered slabs must equal the single-domain run bit for
bit, and the rank-ordered diagnostics must match it.  Self-skips on boxes with fewer than 2 GPUs
(the single-GPU path of the same schedule is covered by the loopback tests)."""
import multiprocessing as mp

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _n_gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _rank_main(rank, nranks, uid, pdict, steps, q):
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2312_05410_b200 import pf
    p = pf.pf_default_params(4)
    for k, v in pdict.items():
        setattr(p, k, v)
    p.device = rank
    with pf.Simulation(p, ("slab", rank, nranks, uid)) as s:
        s.step(steps)
        q.put((rank, s.fields(0), s.diagnostics(0)))


@pytest.mark.skipif(_n_gpus() < 2, reason="needs 2 GPUs (one NCCL rank each)")
@pytest.mark.parametrize("overlap,transport", [(1, 0), (0, 0), (1, 1), (0, 1)])
def test_two_rank_nccl_slabs_equal_single_domain(overlap, transport):
    """transport 0: NCCL send/recv per stage; 1: B11 peer stores into the neighbour's ghost rows
    through CUDA-IPC mappings (handles exchanged over the NCCL communicator) + arrival counters."""
    from paper_2312_05410_b200 import pf
    pdict = dict(nx=512, ny=256, ic_height=64.0, overlap_halo=overlap, graph_steps=0, check_every=10,
                 halo_transport=transport)
    p = pf.pf_default_params(4)
    for k, v in pdict.items():
        setattr(p, k, v)
    steps = 25
    with pf.Simulation(p) as s:
        s.step(steps)
        ref = s.fields(0)
        dref = s.diagnostics(0)
    uid = pf.pf_nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, uid, pdict, steps, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict((r, (f, d)) for r, f, d in (q.get(timeout=300) for _ in procs))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for fld in range(3):
        got = np.concatenate([out[0][0][fld], out[1][0][fld]], axis=0)
        assert np.array_equal(got, ref[fld]), fld
    for r in range(2):   # diagnostics are gathered over ranks and summed in rank order
        np.testing.assert_allclose(out[r][1][:4], dref[:4], rtol=1e-12, atol=0)
