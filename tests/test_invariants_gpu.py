"""GPU-only invariants of the CUDA path (bitwise): kernel paths agree, x-translation equivariance,
ensemble member == single run, run-to-run determinism, resume == straight run, loopback y-slabs ==
single domain, CUDA graphs == direct launches; blow-up detection."""
import numpy as np
import pytest

from paper_2312_05410_b200 import pf
from tests import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pf.lib()


def _base(nx=96, ny=48, **kw):
    p = pf.pf_default_params(2).replace(nx=nx, ny=ny, ic_height=ny / 4, graph_steps=0, seed=21,
                                       theta_deg=71.0, M_A_bulk=12.0, M_B_bulk=6.0, M_A_surf=9.0,
                                       M_B_surf=3.0)
    return p.replace(**kw)


def _run(p, n, mode="single", init=None):
    with pf.Simulation(p, mode) as s:
        if init is not None:
            for m, u in enumerate(init):
                s.set_fields(m, *u)
        s.step(n)
        return [s.fields(m) for m in range(p.n_members)]


def _eq(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("nx,ny,members", [(64, 64, 1), (96, 48, 2), (260, 40, 1), (512, 72, 2), (16, 20, 1),
                                            (1000, 24, 1), (4096, 12, 1)])
def test_tile_stream_pair_paths_bitwise(nx, ny, members):
    """The stage kernels (tile; pair streaming) give identical bits: same per-cell arithmetic, so
    any difference is an indexing, ring-refill or ghost-frame bug.  Covers one to four compute warps
    per strip, several strips with a ragged last strip and minimal grids."""
    p = _base(nx, ny, n_members=members, rate_lo=0.5, rate_hi=2.0)
    a = _run(p.replace(kernel_path=1), 20)
    c = _run(p.replace(kernel_path=3), 20)
    for m in range(members):
        assert _eq(a[m], c[m]), m


@pytest.mark.parametrize("nx,ny,members,extra", [(64, 64, 1, {}), (512, 72, 2, {}), (1000, 24, 1, {}),
                                                  (260, 40, 2, dict(mob_lo=0.5, mob_hi=1.0)),
                                                  (128, 40, 2, dict(fe_model=1, omega=2.2, temp_rs=0.45, dt=4e-4))])
def test_fp32_pair_kernel_bitwise(nx, ny, members, extra):
    """fp32 storage (configs[4]'s precision): the pair kernel computes a lane's two cells as one
    packed pair (FADD2 / FMUL2 / FFMA2) and must still give the scalar tile kernel's bits."""
    p = _base(nx, ny, n_members=members, rate_lo=0.5, rate_hi=2.0, precision=pf.PF_F32, **extra)
    a = _run(p.replace(kernel_path=1), 20)
    c = _run(p.replace(kernel_path=3), 20)
    for m in range(members):
        assert _eq(a[m], c[m]), m


@pytest.mark.parametrize("shift", [64, 5, 1])
def test_x_translation_equivariance(shift):
    nx, ny = 256, 40
    p = _base(nx, ny, ic=pf.PF_IC_NONE)
    u = inputs.random_state(nx, ny, 5, phi_kind="smooth")
    a = _run(p, 15, init=[u])[0]
    us = [np.roll(f, shift, axis=1) for f in u]
    b = _run(p, 15, init=[us])[0]
    for fa, fb in zip(a, b):
        assert np.array_equal(np.roll(fa, shift, axis=1), fb)


def test_member_equals_single_run():
    p = _base(128, 40, n_members=4, rate_lo=0.5, rate_hi=2.0)
    ens = _run(p, 12)
    for m in (0, 3):
        single = _run(p.replace(n_members=1, member_offset=m), 12)[0]
        assert _eq(ens[m], single), m


def test_run_to_run_determinism_and_diagnostics():
    p = _base(192, 64, n_members=2)
    with pf.Simulation(p) as s1, pf.Simulation(p) as s2:
        s1.step(30); s2.step(30)
        for m in range(2):
            assert _eq(s1.fields(m), s2.fields(m))
            assert np.array_equal(s1.diagnostics(m), s2.diagnostics(m))


def test_resume_equals_straight_run():
    p = _base(128, 48)
    straight = _run(p, 40)[0]
    with pf.Simulation(p) as s:
        s.step(17)
        u = s.fields(0)
        st, t, _, _ = s.info()
    with pf.Simulation(p.replace(ic=pf.PF_IC_NONE)) as s:
        s.set_fields(0, *u)
        pf.pf_set_time(s.ctx, st, t)
        s.step(23)
        assert _eq(s.fields(0), straight)
        assert s.info()[0] == 40


@pytest.mark.parametrize("nslabs,path,overlap,graph", [(2, 0, 1, 0), (4, 0, 1, 0), (4, 1, 1, 0), (8, 0, 1, 0),
                                                        (4, 3, 1, 0), (4, 0, 0, 0), (2, 0, 1, 8), (16, 0, 1, 0)])
def test_loopback_slabs_equal_single_domain(nslabs, path, overlap, graph):
    """The y-slab decomposition (2-row halo exchanged after every stage) is bitwise invisible, with
    and without the overlap schedule (boundary bands first, exchange on the comm stream while the
    interior is updated), inside CUDA graphs, and for slabs of 4 rows (no overlap possible)."""
    p = _base(128, 64, n_members=2, kernel_path=path, overlap_halo=overlap, graph_steps=graph)
    a = _run(p, 25)
    b = _run(p, 25, mode=("loopback", nslabs))
    for m in range(2):
        assert _eq(a[m], b[m]), m
    with pf.Simulation(p, ("loopback", nslabs)) as s:
        s.step(3)
        d = s.diagnostics(1)
    with pf.Simulation(p) as s:
        s.step(3)
        d1 = s.diagnostics(1)
    np.testing.assert_allclose(d, d1, rtol=1e-12, atol=0)


@pytest.mark.parametrize("nslabs,path,overlap,prec", [(2, 0, 1, 0), (4, 0, 1, 0), (8, 3, 1, 0), (4, 0, 0, 0),
                                                       (16, 0, 1, 0), (4, 3, 1, 1), (3, 1, 1, 0)])
def test_loopback_peer_transport_equals_single_domain(nslabs, path, overlap, prec):
    """B11 (halo_transport = 1): the push kernel stores each slab's 2 boundary rows straight into
    the neighbours' ghost rows and bumps their arrival counters, the receiving stream waits on the
    counters (cuStreamWaitValue32) -- bitwise the single-domain run (fp64 and fp32, with and
    without the overlap schedule, 4-row slabs), diagnostics too, and a pf_set_fields resume
    (which re-exchanges the halo through the same path) continues bitwise."""
    p = _base(128, 48 * nslabs if nslabs == 3 else 64, n_members=2, kernel_path=path, overlap_halo=overlap,
              graph_steps=8, precision=prec)
    a = _run(p, 25)
    q = p.replace(halo_transport=1)
    b = _run(q, 25, mode=("loopback", nslabs))
    for m in range(2):
        assert _eq(a[m], b[m]), m
    with pf.Simulation(q, ("loopback", nslabs)) as s:
        s.step(11)
        u = s.fields(1)
        d = s.diagnostics(1)
    with pf.Simulation(p) as s:
        s.step(11)
        d1 = s.diagnostics(1)
    np.testing.assert_allclose(d, d1, rtol=1e-12 if prec == 0 else 1e-6, atol=0)
    with pf.Simulation(q.replace(ic=pf.PF_IC_NONE), ("loopback", nslabs)) as s:
        s.set_fields(1, *u)
        s.step(14)
        assert _eq(s.fields(1), a[1])


@pytest.mark.parametrize("nslabs,path,overlap,prec", [(2, 0, 1, 0), (4, 0, 1, 0), (8, 3, 0, 0), (4, 1, 1, 1),
                                                       (16, 0, 1, 0)])
def test_loopback_nccl_self_transport_equals_single_domain(nslabs, path, overlap, prec):
    """halo_transport = 2: the slabs of a one-GPU context exchange their boundary rows through a
    1-rank NCCL communicator (ncclSend to self matched with ncclRecv from self, one group per
    exchange), i.e. through the issue code of the multi-rank NCCL transport (nccl_rows), and the
    diagnostics go through ncclAllGather -- bitwise the single-domain run (fp64 and fp32, with and
    without the overlap schedule, 4-row slabs), and a pf_set_fields resume continues bitwise."""
    p = _base(128, 64, n_members=2, kernel_path=path, overlap_halo=overlap, precision=prec)
    a = _run(p, 25)
    q = p.replace(halo_transport=2)
    b = _run(q, 25, mode=("loopback", nslabs))
    for m in range(2):
        assert _eq(a[m], b[m]), m
    with pf.Simulation(q, ("loopback", nslabs)) as s:
        s.step(11)
        u = s.fields(1)
        d = s.diagnostics(1)
    with pf.Simulation(p) as s:
        s.step(11)
        d1 = s.diagnostics(1)
    np.testing.assert_allclose(d, d1, rtol=1e-12 if prec == 0 else 1e-6, atol=0)
    with pf.Simulation(q.replace(ic=pf.PF_IC_NONE), ("loopback", nslabs)) as s:
        s.set_fields(1, *u)
        s.step(14)
        assert _eq(s.fields(1), a[1])


def test_nccl_self_transport_inside_cuda_graphs_bitwise():
    """PF_NCCL_SELF_GRAPH=1 (read once per process, hence the subprocess): the NCCL groups of
    transport 2 captured into the step graphs give the bits of the direct launches."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np\n"
        "from paper_2312_05410_b200 import pf\n"
        "p = pf.pf_default_params(2).replace(nx=128, ny=64, ic_height=16.0, n_members=2, seed=21, halo_transport=2,\n"
        "                                    overlap_halo=1)\n"
        "out = []\n"
        "for g in (0, 8):\n"
        "    with pf.Simulation(p.replace(graph_steps=g), ('loopback', 4)) as s:\n"
        "        s.step(25)\n"
        "        out.append([s.fields(m) for m in range(2)])\n"
        "assert all(np.array_equal(x, y) for a, b in zip(*out) for x, y in zip(a, b))\n"
        "print('graph == direct')\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PF_NCCL_SELF_GRAPH="1"), cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "graph == direct" in r.stdout, (r.stdout[-1000:], r.stderr[-3000:])


def test_nccl_self_transport_is_loopback_only():
    """pf_create_slab (one slab per rank) rejects transport 2; a single domain ignores it."""
    p = _base(64, 64, halo_transport=2)
    with pf.Simulation(p) as s:
        s.step(2)
    with pytest.raises(Exception, match="halo_transport 2"):
        pf.Simulation(p, ("slab", 0, 2, pf.pf_nccl_unique_id()))


def test_loopback_peer_transport_large_grid_cfg4_physics():
    """configs[3] physics on 1024 x 512 in 8 slabs of 64 rows, peer transport: bitwise the
    single domain after 30 steps (interface on a slab boundary)."""
    p = pf.pf_default_params(4).replace(nx=1024, ny=512, ic_height=128.0)
    a = _run(p, 30)
    b = _run(p.replace(halo_transport=1), 30, mode=("loopback", 8))
    assert _eq(a[0], b[0])


def test_loopback_overlap_large_grid_cfg4_physics():
    """A 1024 x 512 grid of configs[3] physics in 4 slabs of 128 rows (interface on a slab
    boundary): overlap schedule bitwise equal to the single domain after 30 steps."""
    p = pf.pf_default_params(4).replace(nx=1024, ny=512, ic_height=128.0)
    a = _run(p, 30)
    b = _run(p, 30, mode=("loopback", 4))
    assert _eq(a[0], b[0])


def test_graphs_equal_direct_launches():
    p = _base(128, 48)
    a = _run(p.replace(graph_steps=0), 60)[0]
    b = _run(p.replace(graph_steps=16), 60)[0]
    assert _eq(a, b)


def test_blowup_detected_and_cleared():
    p = _base(64, 32, check_every=5)
    with pf.Simulation(p) as s:
        c, phi, rho = s.fields(0)
        phi[10, 7] = np.nan
        s.set_fields(0, c, phi, rho)
        with pytest.raises(pf.PfError) as e:
            s.step(12)
        assert e.value.status == pf.PF_ERR_BLOWUP
        assert "phi" in str(e.value) and "(0, 5]" in str(e.value)
        with pytest.raises(pf.PfError) as e:
            s.step(1)
        assert e.value.status == pf.PF_ERR_STATE
        c2, phi2, rho2 = _run(p, 0)[0]
        s.set_fields(0, c2, phi2, rho2)
        s.step(3)
        assert np.all(np.isfinite(s.fields(0)[1]))


def test_get_set_roundtrip_all_members():
    p = _base(128, 32, n_members=3)
    with pf.Simulation(p) as s:
        c, phi, rho = s.fields(-1)
        assert c.shape == (3, 32, 128)
        s.set_fields(-1, c[::-1].copy(), phi[::-1].copy(), rho[::-1].copy())
        c2, _, _ = s.fields(-1)
        assert np.array_equal(c2, c[::-1])


@pytest.mark.parametrize("chunks", [1, 2, 3, 6])
def test_run_host_pipeline_equals_set_step_get(chunks):
    """pf_run_host (uploads / steps / downloads pipelined over member chunks on three streams) is
    bitwise the same as pf_set_fields + pf_step + pf_get_fields, and keeps the step count."""
    p = _base(128, 48, n_members=6, rate_lo=0.5, rate_hi=2.0)
    with pf.Simulation(p) as s:
        c0, p0, r0 = s.fields(-1)
    cin = c0[::-1].copy(); pin = p0[::-1].copy(); rin = r0[::-1].copy()
    with pf.Simulation(p) as s:
        s.set_fields(-1, cin, pin, rin)
        s.step(17)
        want = s.fields(-1)
    with pf.Simulation(p) as s:
        out = [np.empty_like(cin) for _ in range(3)]
        pf.pf_run_host(s.ctx, 17, cin, pin, rin, *out, chunks=chunks)
        assert s.info()[0] == 17
        for a, b in zip(out, want):
            assert np.array_equal(a, b)
        # device state is the result: continuing gives the straight-run result
        pf.pf_run_host(s.ctx, 5, None, None, None, *out, chunks=chunks)
        s2 = pf.Simulation(p)
        s2.set_fields(-1, cin, pin, rin)
        s2.step(22)
        for a, b in zip(out, s2.fields(-1)):
            assert np.array_equal(a, b)
        s2.close()


def test_run_host_blowup():
    p = _base(64, 32, n_members=4)
    with pf.Simulation(p) as s:
        c, phi, rho = s.fields(-1)
        phi[2, 10, 7] = np.nan
        out = [np.empty_like(c) for _ in range(3)]
        with pytest.raises(pf.PfError) as e:
            pf.pf_run_host(s.ctx, 4, c, phi, rho, *out, chunks=2)
        assert e.value.status == pf.PF_ERR_BLOWUP and "first member 2" in str(e.value)


def test_stochastic_inflow_invariants():
    """With stochastic inflow: member == single run (draws keyed by the global member id), loopback
    slabs == single domain, pf_run_host == pf_step, and resuming at step n draws step n's row."""
    p = _base(96, 64, n_members=3, noise_rho=0.25)
    ens = _run(p, 15)
    one = _run(p.replace(n_members=1, member_offset=2), 15)[0]
    assert _eq(ens[2], one)
    b = _run(p, 15, mode=("loopback", 4))
    for m in range(3):
        assert _eq(ens[m], b[m])
    with pf.Simulation(p) as s:
        c, phi, rho = s.fields(-1)
        out = [np.empty_like(c) for _ in range(3)]
        pf.pf_run_host(s.ctx, 15, c, phi, rho, *out, chunks=3)
        for m in range(3):
            assert _eq([out[0][m], out[1][m], out[2][m]], ens[m])
    with pf.Simulation(p) as s:
        s.step(6)
        u = s.fields(-1)
        st, t, _, _ = s.info()
    with pf.Simulation(p.replace(ic=pf.PF_IC_NONE)) as s:
        s.set_fields(-1, *u)
        pf.pf_set_time(s.ctx, st, t)
        s.step(9)
        for m in range(3):
            assert _eq(s.fields(m), ens[m])


def test_regular_solution_paths_bitwise():
    """The regular-solution variant gives identical bits on the tile and pair kernels."""
    p = _base(128, 40, n_members=2, fe_model=1, omega=2.2, temp_rs=0.45, rate_lo=0.5, rate_hi=2.0, dt=4e-4)
    a = _run(p.replace(kernel_path=1), 12)
    c = _run(p.replace(kernel_path=3), 12)
    for m in range(2):
        assert _eq(a[m], c[m])


@pytest.mark.parametrize("nx,ny,members,extra", [(128, 40, 2, {}), (512, 72, 2, {}), (96, 64, 3, dict(noise_rho=0.2)),
                                                  (1000, 24, 1, {}), (200, 48, 2, dict(fe_model=1, omega=2.2,
                                                                                     temp_rs=0.45, dt=4e-4))])
def test_warp_specialised_step_kernel_bitwise(nx, ny, members, extra):
    """The experimental warp-specialised step kernel (kernel_path 5: stage-1 warps hand u* to
    stage-2 warps through a shared-memory ring, one HBM pass per step) gives the same bits as the
    two-stage pair kernel."""
    p = _base(nx, ny, n_members=members, rate_lo=0.5, rate_hi=2.0, **extra)
    a = _run(p.replace(kernel_path=3), 7)
    b = _run(p.replace(kernel_path=5), 7)
    for m in range(members):
        assert _eq(a[m], b[m]), m


@pytest.mark.parametrize("nx,ny,members,extra", [(64, 64, 1, {}), (128, 128, 1, {}), (96, 48, 3, {}), (33, 65, 2, {}),
                                                  (128, 40, 2, dict(mob_lo=0.5, mob_hi=1.0)),
                                                  (80, 32, 1, dict(fe_model=1, omega=2.2, temp_rs=0.45, dt=4e-4)),
                                                  (500, 24, 1, {}), (16, 8, 5, {}), (8, 8, 1, {})])
def test_band_small_grid_kernel_bitwise(nx, ny, members, extra):
    """The band small-grid kernel (kernel_path 6: each member one thread-block cluster of <= 16
    bands of >= 2 rows held in shared memory, halo rows pushed into the neighbours' shared memory,
    all steps of a check interval in one launch) gives the same bits as the tile kernel: uneven
    bands, bands of exactly 2 rows, several members (clusters), per-member mobilities, the
    regular-solution energy, and several launches."""
    p = _base(nx, ny, n_members=members, rate_lo=0.5, rate_hi=2.0, check_every=9, **extra)
    a = _run(p.replace(kernel_path=1), 23)
    b = _run(p.replace(kernel_path=6), 23)
    for m in range(members):
        assert _eq(a[m], b[m]), m


def test_band_kernel_is_the_small_grid_default_and_resumes():
    """The default small-grid paths (configs[0]: band kernel; configs[1]: persistent tile kernel)
    equal the pair kernel bitwise; a band run continues bitwise on the pair kernel (valid ghost
    frame)."""
    for cfg in (1, 2):
        p = pf.pf_default_params(cfg)
        a = _run(p.replace(kernel_path=0, check_every=50), 120)
        b = _run(p.replace(kernel_path=3, graph_steps=0), 120)
        assert _eq(a[0], b[0]), cfg
    p = _base(96, 40, check_every=10)
    with pf.Simulation(p.replace(kernel_path=6)) as s:
        s.step(15)
        u = s.fields(0)
    with pf.Simulation(p.replace(kernel_path=3, ic=pf.PF_IC_NONE)) as s:
        s.set_fields(0, *u)
        s.step(10)
        x = s.fields(0)
    y = _run(p.replace(kernel_path=1), 25)[0]
    assert _eq(x, y)


@pytest.mark.parametrize("nx,ny,members,extra", [(64, 64, 1, {}), (96, 48, 3, {}), (33, 65, 2, {}),
                                                  (128, 40, 2, dict(mob_lo=0.5, mob_hi=1.0)),
                                                  (80, 32, 1, dict(fe_model=1, omega=2.2, temp_rs=0.45, dt=4e-4)),
                                                  (384, 384, 1, {})])   # > 2^17 cells: 32 x 16 tiles
def test_persistent_small_grid_kernel_bitwise(nx, ny, members, extra):
    """The persistent small-grid kernel (kernel_path 7: all steps of a check interval in one
    cooperative launch) gives the same bits as the stage kernels, across several check intervals,
    and leaves a valid ghost frame behind (a later pair-kernel run continues bitwise)."""
    p = _base(nx, ny, n_members=members, rate_lo=0.5, rate_hi=2.0, check_every=9, **extra)
    a = _run(p.replace(kernel_path=1), 23)
    b = _run(p.replace(kernel_path=7), 23)
    for m in range(members):
        assert _eq(a[m], b[m]), m
