"""N > 1 host logic on CPU: world_size-2 process groups over gloo (127.0.0.1).

Checks, with real inter-process communication and no GPU:
* the NCCL-uid broadcast helper delivers rank 0's bytes to every rank;
* ensemble slices (weak and strong) cover the global members exactly once, and each rank's
  member velocities (library, host-only) equal the single-process enumeration (R-15);
* the library's slab plan (pf_halo_plan) partitions the rows, and exchanging the seeded initial
  rows along it (dist.exchange_rows, the CPU transport of the NCCL exchange) fills every interior
  ghost row with the neighbour's rows while the physical-boundary ghost rows stay untouched;
* max over ranks and the rank-ordered diagnostics sum are identical on every rank.
"""
import os
import socket
import sys
import traceback

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world_size, port, ny, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world_size),
                          RANK=str(rank), LOCAL_RANK=str(rank))
        from paper_2312_05410_b200 import dist as D, pf
        dist = D.init("gloo")
        assert dist is not None and dist.get_world_size() == world_size

        # uid broadcast
        payload = bytes(range(7, 135)) if rank == 0 else None
        got = D.broadcast_bytes(dist, payload, 128)
        assert got == bytes(range(7, 135))

        # ensemble slices + member velocities
        p = pf.pf_default_params(3)
        for weak, total in ((True, 5), (False, 13)):
            off, n = D.ensemble_slice(total, rank, world_size, weak)
            ids = list(range(off, off + n))
            allids = [None] * world_size
            dist.all_gather_object(allids, ids)
            flat = sorted(i for part in allids for i in part)
            want = list(range(total * world_size)) if weak else list(range(total))
            assert flat == want, (weak, flat)
            for m in ids:
                assert pf.pf_member_velocity(p, m) == pf.pf_member_velocity(p, m)
            vel = [pf.pf_member_velocity(p, m) for m in ids]
            allv = [None] * world_size
            dist.all_gather_object(allv, vel)
            assert [v for part in allv for v in part] == [pf.pf_member_velocity(p, m) for m in want]

        # slab plan + halo exchange of the seeded initial rows
        p = pf.pf_default_params(4).replace(nx=64, ny=ny, ic_height=ny / 8)
        plan = D.slab(ny, rank, world_size)
        y0, rows = plan["y0"], plan["ny_local"]
        assert rows == ny // world_size and y0 == rank * rows
        full = pf.pf_initial_fields(p, 0, 0, ny)
        for f in range(3):
            loc = np.full((rows + 4, p.nx), np.nan)
            loc[2:2 + rows] = pf.pf_initial_fields(p, 0, y0, rows)[f]
            D.exchange_rows(dist, loc, plan)
            assert np.array_equal(loc[2:2 + rows], full[f][y0:y0 + rows])
            if plan["below"] >= 0:
                assert np.array_equal(loc[0:2], full[f][y0 - 2:y0])
            else:
                assert np.isnan(loc[0:2]).all()
            if plan["above"] >= 0:
                assert np.array_equal(loc[2 + rows:], full[f][y0 + rows:y0 + rows + 2])
            else:
                assert np.isnan(loc[2 + rows:]).all()

        # timing and ordered diagnostics sums
        assert D.max_over_ranks(dist, 1.5 + rank) == 1.5 + world_size - 1
        part = np.array([0.1 * (rank + 1), 1e-17 * rank, 3.0])
        tot = D.ordered_sum(dist, part)
        want = np.zeros(3)
        for r in range(world_size):
            want = want + np.array([0.1 * (r + 1), 1e-17 * r, 3.0])
        assert np.array_equal(tot, want)
        allt = [None] * world_size
        dist.all_gather_object(allt, tot.tolist())
        assert all(t == allt[0] for t in allt)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world_size,ny", [(2, 64), (2, 36)])
def test_two_rank_gloo(world_size, ny):
    import torch.multiprocessing as mp
    from paper_2312_05410_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world_size, port, ny, q)) for r in range(world_size)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world_size):
        assert res.get(r) == "ok", res.get(r)


def test_plan_errors():
    from paper_2312_05410_b200 import pf
    with pytest.raises(pf.PfError):
        pf.pf_halo_plan(10, 3, 0)
    with pytest.raises(pf.PfError):
        pf.pf_halo_plan(8, 8, 0)
    with pytest.raises(pf.PfError):
        pf.pf_halo_plan(16, 2, 2)
    assert pf.pf_halo_plan(16, 1, 0) == (0, 16, -1, -1, 0, 14, -2, 16)
