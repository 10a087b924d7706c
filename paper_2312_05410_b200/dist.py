"""Process-group plumbing for N > 1 GPUs (one process per GPU).

torch.distributed is used only to move bytes between the processes: the NCCL unique id that
pf_create_slab needs, per-rank timings (max over ranks) and diagnostics partials (gathered and
summed in rank order, so the result does not depend on reduction order).  The y-slab plan comes
from the library (pf_halo_plan) -- the same plan its NCCL exchange follows -- and
``exchange_rows`` applies that plan to host arrays over any backend (gloo on CPU in the tests), so
the message schedule of the multi-GPU path is exercised without GPUs.  No model arithmetic here.
"""
from __future__ import annotations

import os

import numpy as np

from . import pf


def world():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, device=None):
    """Initialise the default process group when WORLD_SIZE > 1; returns torch.distributed or None."""
    ws, _, _ = world()
    if ws <= 1:
        return None
    import torch.distributed as dist
    if not dist.is_initialized():
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, **kw)
    return dist


def _dev(dist, device):
    import torch
    if device is not None:
        return device
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def broadcast_bytes(dist, data: bytes | None, n: int, src: int = 0, device=None) -> bytes:
    """Rank `src`'s n bytes on every rank (e.g. the 128-byte NCCL unique id)."""
    import torch
    dev = _dev(dist, device)
    t = torch.zeros(n, dtype=torch.uint8, device=dev)
    if dist.get_rank() == src:
        t.copy_(torch.tensor(list(data), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def nccl_uid(dist, device=None) -> bytes:
    """pf_nccl_unique_id on rank 0, broadcast to all ranks."""
    uid = pf.pf_nccl_unique_id() if dist.get_rank() == 0 else None
    return broadcast_bytes(dist, uid, 128, 0, device)


def ensemble_slice(members: int, rank: int, world_size: int, weak: bool = True):
    """(member_offset, n_members) of rank `rank`.  Weak scaling: `members` per rank, global ids
    [rank * members, (rank + 1) * members).  Strong scaling: `members` in total, split into
    contiguous, near-equal slices (R-15 keys seeds and rates by the global id, so the union of the
    slices is the same ensemble for any world size)."""
    if weak:
        return rank * members, members
    lo = members * rank // world_size
    hi = members * (rank + 1) // world_size
    return lo, hi - lo


def slab(ny: int, rank: int, world_size: int) -> dict:
    """The library's y-slab plan of this rank (pf_halo_plan) as a dict."""
    keys = ("y0", "ny_local", "below", "above", "send_down", "send_up", "recv_below", "recv_above")
    return dict(zip(keys, pf.pf_halo_plan(ny, world_size, rank)))


def max_over_ranks(dist, value: float, device=None) -> float:
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_dev(dist, device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ordered_sum(dist, values: np.ndarray, device=None) -> np.ndarray:
    """Sum of every rank's `values` taken in rank order (all-gather, then a fixed-order sum):
    bitwise identical on every rank and for every run with the same world size."""
    import torch
    dev = _dev(dist, device)
    t = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64), device=dev)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    acc = np.zeros_like(np.asarray(values, dtype=np.float64))
    for p_ in parts:
        acc = acc + p_.cpu().numpy()
    return acc


def exchange_rows(dist, field: np.ndarray, plan: dict) -> None:
    """Apply the slab plan to a host array `field` of shape (ny_local + 4, nx) holding local rows
    -2 .. ny_local+1: send the 2 boundary rows to each neighbour and receive its rows into the
    ghost rows, in place (the CPU transport of the library's NCCL exchange)."""
    import torch
    o = 2   # storage row of local row 0
    ops = []
    bufs = []
    if plan["below"] >= 0:
        s = torch.from_numpy(np.ascontiguousarray(field[o + plan["send_down"]:o + plan["send_down"] + 2]))
        r = torch.empty_like(s)
        ops += [dist.P2POp(dist.isend, s, plan["below"]), dist.P2POp(dist.irecv, r, plan["below"])]
        bufs.append((plan["recv_below"], r))
    if plan["above"] >= 0:
        s = torch.from_numpy(np.ascontiguousarray(field[o + plan["send_up"]:o + plan["send_up"] + 2]))
        r = torch.empty_like(s)
        ops += [dist.P2POp(dist.isend, s, plan["above"]), dist.P2POp(dist.irecv, r, plan["above"])]
        bufs.append((plan["recv_above"], r))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for row, r in bufs:
        field[o + row:o + row + 2] = r.numpy()
