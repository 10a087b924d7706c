"""Benchmark of the B200-native PVD phase-field midpoint step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3|4|1|2|5] [--impl ours|reference]

Default workload (N=1 and per rank under torchrun): BASELINE.json configs[2], the ensemble of 64
independent 512 x 512 fp64 members, weak-scaled (64 members per GPU, member ids keyed by rank, no
collective on the step path; R-20).  A "step" is one explicit-midpoint time step of every member:
stage-1 and stage-2 fused kernels, plus the diagnostics / blow-up check every check_every = 100
steps and at the end of the timed call (rows a1-a6 of SURVEY 8(a)).  --config 4 runs the y-slab
decomposition of configs[3] (4096 x 4096*N, NCCL halo exchange per stage).

Rank 0 prints one JSON line.  The oracle (oracle/, test infrastructure) is only executed in the
cpu_baseline leg and under --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/sec and achieved HBM GB/s (fraction of B200 peak) at 1/2/4/8 GPUs"
UNIT = "cell-updates/s"
# Algorithmic HBM bytes per cell and launch of the stage kernel: stage 1 reads
# u^n (3 fields) and writes u* (3 fields); stage 2 reads u* and u^n (6) and writes u^{n+1} (3).
VALUES_STAGE1, VALUES_STAGE2 = 6, 9


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(config_key):
    """Per-launch dram bytes of the stage kernel from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(config_key)
    except Exception:
        return None


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML during the timed region."""

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_member_worker(cfg, member, warmup, steps, seconds, out):
    """One oracle process (single thread): `warmup` untimed steps of member `member` of configs[cfg -
    1] (a 512 x 512 tile for the single-grid configs), then `steps` timed steps (or as many as fit
    in `seconds` when steps is 0).  Puts (cells, steps, seconds) on `out`."""
    sys.path.insert(0, ROOT)
    from oracle import oracle as ora
    pr = ora.preset(cfg)
    m = ora.member_model(pr, member if cfg == 3 else 0)
    nx = PRESETS[cfg][0]
    tx = min(512, nx)
    if cfg == 3:
        u = ora.initial_fields(pr["ic"], nx, PRESETS[cfg][1], member)
    else:
        c, phi, rho = ora.initial_fields_rows(pr["ic"], nx, 0, 0, min(512, PRESETS[cfg][1]))
        u = (c[:, :tx].copy(), phi[:, :tx].copy(), rho[:, :tx].copy())
    cells = u[0].size
    if warmup:
        u = ora.step(m, *u, warmup)
    done, t0 = 0, time.perf_counter()
    if steps > 0:
        u = ora.step(m, *u, steps)
        done = steps
    else:
        while time.perf_counter() - t0 < seconds:
            u = ora.step(m, *u, 1)
            done += 1
    out.put((cells, done, time.perf_counter() - t0))


def _oracle_ensemble(cfg, procs, warmup, steps, seconds=0.0):
    """The oracle as it stands on `procs` concurrent single-threaded processes (one ensemble member,
    or one 512 x 512 tile, each; SURVEY 8(d) "min(nproc, members) concurrent oracle processes").
    Returns (cells per step over all processes, steps, wall seconds of the slowest process)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")            # the parent may hold a CUDA context: never fork it
    q = ctx.Queue()
    ps = [ctx.Process(target=_oracle_member_worker, args=(cfg, k, warmup, steps, seconds, q)) for k in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    cells = sum(r[0] for r in res)
    nsteps = min(r[1] for r in res)
    wall = max(r[2] for r in res)
    return cells, nsteps, wall, res


def _cpu_baseline(seconds=12.0):
    """The oracle as it stands on min(nproc, 64) concurrent single-threaded processes, one member of
    configs[2] (512 x 512 fp64) each, for ~`seconds`: aggregate cell-updates/s of the host."""
    procs = min(os.cpu_count() or 1, PRESETS[3][2])
    cells, nsteps, wall, res = _oracle_ensemble(3, procs, 0, 0, seconds)
    value = sum(r[0] * r[1] / r[2] for r in res)
    return {"value": value, "unit": UNIT, "cores": procs, "kind": "oracle", "cpu_model": _cpu_model(),
            "nproc": os.cpu_count(),
            "sample": f"configs[2] members 0..{procs - 1} (512x512 fp64), one single-threaded oracle process per "
                      f"member on {procs} cores concurrently, {min(r[1] for r in res)}-{max(r[1] for r in res)} "
                      f"midpoint steps each in {wall:.1f} s; value = sum of the per-process rates"}


# (nx, ny, members, storage) of BASELINE.json configs[0..4] (R-13, R-14)
PRESETS = {1: (64, 64, 1, "fp64"), 2: (256, 256, 1, "fp64"), 3: (512, 512, 64, "fp64"),
           4: (4096, 4096, 1, "fp64"), 5: (8192, 8192, 1, "fp32")}


def workload_config(cfg, ws):
    """The `config` object of the JSON line (identical for both arms)."""
    nx, ny, mem, dt = PRESETS[cfg]
    esz = 8 if dt == "fp64" else 4
    if cfg == 3:
        desc = f"configs[2]: {mem} x {nx}x{ny} {dt} ensemble per GPU (weak, {mem * ws} members total)"
    elif cfg == 4:
        ny = ny * ws
        desc = f"configs[3]: {nx}x{ny} {dt} y-slab decomposed over {ws} GPU(s) (weak: 4096 rows per GPU)"
    elif cfg == 5:
        desc = f"configs[4]: {nx}x{ny} {dt} y-slab decomposed over {ws} GPU(s) (strong)"
    else:
        desc = f"configs[{cfg - 1}]: {mem} x {nx}x{ny} {dt}"
    cells = mem * nx * ny // (ws if cfg == 5 else 1) // (ws if cfg == 4 else 1)
    l2 = f"state {2 * 3 * cells * esz / 2**20:.0f} MiB per GPU " + (
        "(inputs larger than L2)" if 2 * 3 * cells * esz > 126 * 2**20 else "(L2-resident; no flush)")
    return {"workload": desc, "nx": nx, "ny": ny, "members_per_gpu": mem, "check_every": 100, "l2": l2}


def run_reference(args):
    """--impl reference: the oracle (the reference arm of this tier) as it stands, on the host cores:
    min(nproc, members) concurrent single-threaded processes, each advancing one ensemble member
    (configs[2]) or one 512 x 512 tile (the single-grid configs) through W warm-up and K timed
    explicit-midpoint steps.  A "step" of this arm is therefore one step of that bounded sample;
    ms_per_step is its measured wall time per step (not extrapolated)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = args.config
    members = PRESETS[cfg][2] * (ws if cfg == 3 else 1)
    procs = max(1, min(os.cpu_count() or 1, members if cfg == 3 else 1))
    cells, nsteps, wall, res = _oracle_ensemble(cfg, procs, args.warmup, args.steps)
    v = cells * nsteps / wall
    cfgd = workload_config(cfg, ws)
    sample = (f"{procs} concurrent single-threaded oracle processes ({_cpu_model()}, nproc {os.cpu_count()}), each "
              f"{'one member (512x512 fp64) of' if cfg == 3 else 'a 512x512 fp64 tile of'} configs[{cfg - 1}]: "
              f"{args.warmup} warm-up + {nsteps} timed midpoint steps in {wall:.2f} s (slowest process)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": nsteps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / nsteps,
            "higher_is_better": True, "scaling": "strong" if cfg == 5 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded BASELINE.json configs recipe, DESIGN.md 5)", "config": cfgd,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": procs, "kind": "oracle", "cpu_model": _cpu_model(),
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _timed_steps(sim, stream, steps, dist, dev):
    """Device time (ms, max over ranks) of one pf_step(steps) call, CUDA events on the ctx stream,
    barrier + synchronize on both sides."""
    import torch
    from paper_2312_05410_b200 import dist as D

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sim.step(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    return D.max_over_ranks(dist, ms, dev) if dist is not None else ms


def _slab_leg(args, ws, rank, local, dist, dev):
    """The y-slab path of configs[3] at the same N: weak-scaled 4096 x (4096 N) fp64,
    4096 rows per GPU, the 2-row halo exchanged per stage over NCCL (pf_create_slab) and overlapped
    with the interior update; timed like the main line (K steps after W warm-up, max over ranks).
    At N > 1 rank 0 also times the single-GPU 4096^2 domain (the other ranks wait), so the weak-
    scaling efficiency T(1)/T(N) of this run is reported next to the per-GPU rate."""
    import torch
    from paper_2312_05410_b200 import dist as D
    from paper_2312_05410_b200 import pf
    p = pf.pf_default_params(4).replace(device=local)
    p = p.replace(ny=p.ny * ws, halo_transport=1 if args.slab_transport == "peer" else 0)
    mode = ("slab", rank, ws, D.nccl_uid(dist, dev)) if ws > 1 else "single"
    with pf.Simulation(p, mode) as sim:
        stream = torch.cuda.ExternalStream(pf.pf_stream(sim.ctx), device=dev)
        sim.step(args.warmup)
        ms = _timed_steps(sim, stream, args.steps, dist, dev)
        cells_local = p.nx * sim.ny_local
    ms1 = ms
    if ws > 1:
        if rank == 0:
            p1 = pf.pf_default_params(4).replace(device=local)
            with pf.Simulation(p1) as s1:
                st1 = torch.cuda.ExternalStream(pf.pf_stream(s1.ctx), device=dev)
                s1.step(args.warmup)
                ms1 = _timed_steps(s1, st1, args.steps, None, dev)
        if dist is not None:
            dist.barrier()
    if rank != 0:
        return None
    loop = None
    if ws == 1:
        # One GPU has no neighbour: time the slab SCHEDULE instead -- the same 4096^2 domain as 2
        # loopback y-slabs on this GPU whose 2-row halos go through NCCL (sends to self on a 1-rank
        # communicator, halo_transport 2: the multi-rank transport's issue code) overlapped with
        # the interior update.  Same cells per step as the single domain above.
        q = pf.pf_default_params(4).replace(device=local, halo_transport=2, overlap_halo=1, graph_steps=0)
        with pf.Simulation(q, ("loopback", 2)) as s2:
            st2 = torch.cuda.ExternalStream(pf.pf_stream(s2.ctx), device=dev)
            s2.step(args.warmup)
            l0 = pf.pf_launch_count(s2.ctx)
            runs2 = [_timed_steps(s2, st2, args.steps, None, dev) for _ in range(5)]
            ms2 = sorted(runs2)[2]
            l1 = l0 + (pf.pf_launch_count(s2.ctx) - l0) // 5
        loop = {"workload": "the same 4096 x 4096 domain as 2 loopback y-slabs of 2048 rows on this GPU, 2-row halo "
                            "per stage over NCCL (ncclSend/ncclRecv to self, 1-rank communicator) overlapped with "
                            "the interior update",
                "value": q.nx * q.ny * args.steps / (ms2 * 1e-3), "unit": UNIT, "ms_per_step": ms2 / args.steps,
                "schedule_efficiency": ms / ms2, "launches": l1 - l0,
                "runs_ms_per_step": [r / args.steps for r in runs2],
                "timing": "median of 5 timed calls of K steps (a call now and then takes 2-8x longer on the "
                          "host side of NCCL's group launches; profiles/r2/nccl_self_bench_r2t3.jsonl)",
                "halo_bytes_per_stage_per_neighbour": 2 * 3 * (q.nx + 8) * 8}
    value = cells_local * ws * args.steps / (ms * 1e-3)
    out = _slab_line(args, p, ws, cells_local, value, ms, ms1)
    if loop is not None:
        out["loopback_nccl"] = loop
    return out


def _slab_line(args, p, ws, cells_local, value, ms, ms1):
    return {"workload": f"configs[3] weak: {p.nx} x {p.ny} fp64 in {ws} y-slab(s) of {cells_local // p.nx} rows, "
                        + (("2-row halo per stage over NCCL (ncclSend/Recv on a comm stream)"
                            if args.slab_transport == "nccl" else
                            "2-row halo per stage as peer stores into the neighbours' ghost rows (B11: CUDA-IPC "
                            "mappings, push kernel + arrival counters)") + " overlapped with the interior update"
                           if ws > 1 else "single domain (no exchange at N = 1)"),
            "value": value, "unit": UNIT, "per_gpu": value / ws, "ms_per_step": ms / args.steps,
            "ms_per_step_1gpu": ms1 / args.steps, "weak_efficiency": ms1 / ms, "steps": args.steps,
            "halo_bytes_per_stage_per_neighbour": 2 * 3 * (p.nx + 8) * 8 if ws > 1 else 0}


_JSON_OUT = sys.stdout


def run_ours(args):
    import numpy as np
    import torch
    from paper_2312_05410_b200 import pf

    from paper_2312_05410_b200 import dist as D
    ws, rank, local = D.world()
    # NCCL (and any other library) may print to stdout -- at NCCL_DEBUG=VERSION its version line goes
    # there whatever NCCL_DEBUG_FILE says, and the N = 1 run creates a communicator too (loopback slab
    # leg): keep the process's fd 1 for the one JSON line and point everything else at stderr.
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if ws > 1:   # NCCL init lines (rank counts of every communicator) go to stderr for the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.gpus != ws and ws > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = D.init("nccl", dev)

    cfg = args.config
    p = pf.pf_default_params(cfg).replace(device=local)
    if cfg == 3:
        off, n = D.ensemble_slice(p.n_members, rank, ws, weak=True)   # weak: 64 members per GPU
        p = p.replace(member_offset=off, n_members=n)
        mode = "single"
        workload = f"configs[2]: {p.n_members} x {p.nx}x{p.ny} fp64 ensemble per GPU (weak, {p.n_members * ws} members total)"
    elif cfg == 4 or cfg == 5:
        p = p.replace(ny=p.ny * ws) if cfg == 4 else p          # cfg4 weak: 4096 x 4096 per GPU
        mode = ("slab", rank, ws, D.nccl_uid(dist, dev)) if ws > 1 else "single"
        workload = (f"configs[{cfg - 1}]: {p.nx}x{p.ny} {'fp64' if p.precision == 0 else 'fp32'}"
                    f" y-slab decomposed over {ws} GPU(s)")
    else:
        mode = "single"
        workload = f"configs[{cfg - 1}]: {p.n_members} x {p.nx}x{p.ny}"
    sim = pf.Simulation(p, mode)
    ctx = sim.ctx
    stream = torch.cuda.ExternalStream(pf.pf_stream(ctx), device=torch.device("cuda", local))
    cells_local = p.n_members * sim.ny_local * p.nx
    esz = 8 if p.precision == pf.PF_F64 else 4

    # warm-up (untimed)
    sim.step(args.warmup)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: K steps through one pf_step(K) call, CUDA events on the ctx stream ----
    l0 = pf.pf_launch_count(ctx)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        sim.step(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = pf.pf_launch_count(ctx) - l0
    ms_max = D.max_over_ranks(dist, ms, dev) if dist is not None else ms
    value = cells_local * ws * args.steps / (ms_max * 1e-3)

    # ---- roofline pass: the same K steps again with every stage launch bracketed by CUDA events
    # on the ctx stream (kept out of the value: the per-launch events add ~2% of gaps) ----
    pf.pf_profile(ctx, True)
    barrier()
    sim.step(args.steps)
    torch.cuda.synchronize()
    prof = pf.pf_profile_read(ctx)
    pf.pf_profile(ctx, False)
    n1, n2 = prof[1], prof[3]
    stage_ms = prof[0] + prof[2]
    nslab_launch = max(1.0, (n1 + n2))
    alg_bytes = cells_local * esz * (VALUES_STAGE1 * n1 + VALUES_STAGE2 * n2)
    achieved_bracketed = alg_bytes / (stage_ms * 1e-3) / 1e9 if stage_ms > 0 else None
    # the stage kernels' average launch duration IN the timed region: the timed region holds the
    # 2K stage launches (back to back, programmatic dependent launch) and the diagnostics launches
    # of the blow-up checks; the latter's event time comes from the bracketed pass.  (Bracketing
    # every stage launch with events breaks the dependent-launch overlap, which makes the
    # bracketed launches 3-7% slower than in the timed step: reported beside, as achieved_bracketed.)
    diag_ms = prof[4] if prof[5] > 0 else 0.0
    stage_ms_live = ms - diag_ms
    achieved = alg_bytes / (stage_ms_live * 1e-3) / 1e9 if stage_ms_live > 0 else achieved_bracketed
    peak, peak_src = _peaks()
    key = f"cfg{cfg}_n{ws}"
    tr = _traffic(key)

    # ---- e2e: the public API with HOST buffers (pinned), copies inside the timed region ----
    hc = torch.empty((p.n_members, sim.ny_local, p.nx), dtype=torch.float64, pin_memory=True)
    hp = torch.empty_like(hc).pin_memory()
    hr = torch.empty_like(hc).pin_memory()
    pf.pf_get_fields(ctx, -1, hc, hp, hr)
    e2e_steps = args.steps
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    oc, op_, orr = (torch.empty_like(hc).pin_memory() for _ in range(3))
    chunks = min(2, p.n_members)   # tools/e2e_chunks.py: 2 even chunks (34.3 G) ~ 3 tapered (34.5 G), steadier
    # one untimed call (creates the copy streams and events), then three timed calls, median
    # reported: the host<->device copies share the node's PCIe / memory bandwidth, which made single
    # e2e samples vary by up to ~30%
    pf.pf_run_host(ctx, 1, hc, hp, hr, oc, op_, orr, chunks)
    torch.cuda.synchronize()
    runs = []
    for _ in range(3):
        e0.record(stream)
        pf.pf_run_host(ctx, e2e_steps, hc, hp, hr, oc, op_, orr, chunks)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_run = e0.elapsed_time(e1)
        if dist is not None:
            ms_run = D.max_over_ranks(dist, ms_run, dev)
        runs.append(ms_run)
    ms_e2e = statistics.median(runs)
    host_bytes = 3 * cells_local * 8
    e2e = {"value": cells_local * ws * e2e_steps / (ms_e2e * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": host_bytes / e2e_steps, "d2h_bytes_per_step": host_bytes / e2e_steps,
           "note": f"pf_run_host: upload of every member from pinned fp64 host buffers, {e2e_steps} steps, "
                   f"download of every member; pipelined over {chunks} member chunks (H2D / compute / D2H "
                   "streams); copies amortised over the steps of one call; one warm-up call, median of 3 timed calls",
           "runs_ms": runs}

    slab = None
    if cfg == 3 and not args.no_slab:
        try:   # a failure of the slab leg (its own NCCL communicator) must not cost the main line
            slab = _slab_leg(args, ws, rank, local, dist, dev)
        except Exception as exc:   # noqa: BLE001 -- reported in the line, not swallowed
            slab = {"error": f"{type(exc).__name__}: {exc}"[:300]} if rank == 0 else None

    line = None
    if rank == 0:
        alg_per_cell_step = esz * (VALUES_STAGE1 + VALUES_STAGE2)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if cfg == 5 else "weak", "vs_baseline": None,
            "dtype": "f64" if p.precision == pf.PF_F64 else "f32",
            "data": "synthetic (seeded BASELINE.json configs recipe, DESIGN.md 5)",
            "config": workload_config(cfg, ws),
            "hbm_gbs_effective": value * alg_per_cell_step / ws / 1e9,
            "hbm_frac_effective": value * alg_per_cell_step / ws / 1e9 / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": tr,
                         "kernel": "pair_kernel (both midpoint stages; stage 1 and stage 2 launches)",
                         "algorithmic_bytes_per_launch": alg_bytes / nslab_launch,
                         "avg_launch_ms": stage_ms_live / nslab_launch,
                         "timing": "stage kernels' share of the timed region: (timed ms - diagnostics ms) / "
                                   "stage launches, CUDA events on the ctx stream",
                         "achieved_bracketed": achieved_bracketed,
                         "avg_launch_ms_bracketed": stage_ms / nslab_launch,
                         "diag_ms": diag_ms, "stage_launches": nslab_launch,
                         "step_share": (stage_ms / args.steps) / (ms_max / args.steps) if ms_max > 0 else None,
                         "peak_source": peak_src},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if slab is not None:
            line["slab"] = slab
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = _cpu_baseline()
        print(json.dumps(line), file=_JSON_OUT, flush=True)
    sim.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-slab", action="store_true", help="skip the configs[3] y-slab leg of the default run")
    ap.add_argument("--slab-transport", choices=["nccl", "peer"], default="nccl",
                    help="halo transport of the slab leg at N > 1: NCCL send/recv (default) or the B11 peer stores")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
