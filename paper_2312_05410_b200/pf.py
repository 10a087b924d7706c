"""Thin ctypes binding of libpf (include/pf.h): argument marshalling only.

Every step of the hot path runs inside libpf.so (host runtime + sm_100a kernels).  This module
never computes model arithmetic and has no fallback: if the shared library is missing it raises.
Function names mirror the C ABI (``pf_create``, ``pf_step``, ...); ``Simulation`` is a small
convenience wrapper over the same calls.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PF_LIB: an alternative in-tree build of the same library (A/B experiments of compile-time knobs)
LIB_PATH = os.environ.get("PF_LIB") or os.path.join(_HERE, "libpf.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "pf.h")

PF_ABI_VERSION = 7
PF_OK, PF_ERR_ARG, PF_ERR_UNSTABLE_DT, PF_ERR_NOMEM, PF_ERR_CUDA, PF_ERR_NCCL, PF_ERR_BLOWUP, \
    PF_ERR_STATE, PF_ERR_ABI = range(9)
STATUS_NAMES = ["PF_OK", "PF_ERR_ARG", "PF_ERR_UNSTABLE_DT", "PF_ERR_NOMEM", "PF_ERR_CUDA",
                "PF_ERR_NCCL", "PF_ERR_BLOWUP", "PF_ERR_STATE", "PF_ERR_ABI"]
PF_F64, PF_F32 = 0, 1
PF_IC_FILM, PF_IC_ROUGH_SUBSTRATE, PF_IC_COLUMNS, PF_IC_NONE = range(4)


class pf_params(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32), ("nx", C.c_int32), ("ny", C.c_int32),
        ("n_members", C.c_int32), ("member_offset", C.c_int32), ("precision", C.c_int32),
        ("dx", C.c_double), ("dt", C.c_double),
        ("kappa_c", C.c_double), ("kappa_phi", C.c_double), ("W_c", C.c_double), ("W_phi", C.c_double),
        ("M_A_bulk", C.c_double), ("M_B_bulk", C.c_double), ("M_A_surf", C.c_double),
        ("M_B_surf", C.c_double), ("sigma_surf", C.c_double), ("M_phi", C.c_double),
        ("D_rho", C.c_double), ("rho_in", C.c_double), ("v0", C.c_double), ("theta_deg", C.c_double),
        ("rate_lo", C.c_double), ("rate_hi", C.c_double), ("theta_span", C.c_double),
        ("mob_lo", C.c_double), ("mob_hi", C.c_double), ("noise_rho", C.c_double),
        ("fe_model", C.c_int32), ("omega", C.c_double), ("temp_rs", C.c_double),
        ("ic", C.c_int32), ("ic_ncols", C.c_int32),
        ("ic_height", C.c_double), ("ic_amp", C.c_double), ("ic_wavelength", C.c_double),
        ("ic_c0", C.c_double), ("ic_c_lo", C.c_double), ("ic_c_hi", C.c_double),
        ("noise_c", C.c_double), ("noise_phi", C.c_double),
        ("noise_c_gaussian", C.c_int32), ("check_every", C.c_int32),
        ("seed", C.c_uint64), ("device", C.c_int32), ("graph_steps", C.c_int32),
        ("kernel_path", C.c_int32), ("overlap_halo", C.c_int32),
        ("halo_transport", C.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}

    def replace(self, **kw) -> "pf_params":
        q = pf_params()
        C.memmove(C.byref(q), C.byref(self), C.sizeof(self))
        for k, v in kw.items():
            if not hasattr(q, k):
                raise AttributeError(k)
            setattr(q, k, v)
        return q


class PfError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")


_lib = None
_ctx_p = C.c_void_p
_D = C.POINTER(C.c_double)


def lib():
    """Load libpf.so (fails loudly if it was not built: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2312_05410_b200.build`")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER(pf_params)
        i32, i64 = C.c_int32, C.c_int64
        sig = {
            "pf_params_size": (C.c_uint32, []),
            "pf_default_params": (C.c_int, [i32, P]),
            "pf_initial_fields": (C.c_int, [P, i64, i32, i32, _D, _D, _D]),
            "pf_member_velocity": (C.c_int, [P, i64, _D, _D]),
            "pf_dt_limit": (C.c_int, [P, _D]),
            "pf_member_mobility": (C.c_int, [P, i64, _D]),
            "pf_inflow_row": (C.c_int, [P, i64, i64, _D]),
            "pf_create": (C.c_int, [P, C.POINTER(_ctx_p)]),
            "pf_nccl_unique_id": (C.c_int, [C.c_char_p]),
            "pf_create_slab": (C.c_int, [P, i32, i32, C.c_char_p, C.POINTER(_ctx_p)]),
            "pf_create_loopback": (C.c_int, [P, i32, C.POINTER(_ctx_p)]),
            "pf_halo_plan": (C.c_int, [i32, i32, i32, C.POINTER(i32)]),
            "pf_run_host": (C.c_int, [_ctx_p, i64, _D, _D, _D, _D, _D, _D, i32]),
            "pf_trajectory": (C.c_int, [_ctx_p, i32, i64, _D, _D]),
            "pf_trajectory_file": (C.c_int, [_ctx_p, C.c_char_p, i32, i64, i32]),
            "pf_s2_nbins": (i32, [i32, i32]),
            "pf_s2": (C.c_int, [_D, i32, i32, i32, C.c_double, _D, _D, i32]),
            "pf_s2_rel_l2": (C.c_int, [_D, _D, i32, i32, i32, C.c_double, _D]),
            "pf_step": (C.c_int, [_ctx_p, i64]),
            "pf_get_fields": (C.c_int, [_ctx_p, i32, _D, _D, _D]),
            "pf_set_fields": (C.c_int, [_ctx_p, i32, _D, _D, _D]),
            "pf_diagnostics": (C.c_int, [_ctx_p, i32, _D]),
            "pf_info": (C.c_int, [_ctx_p, C.POINTER(i64), _D, C.POINTER(i32), C.POINTER(i32)]),
            "pf_shape": (C.c_int, [_ctx_p, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
            "pf_set_time": (C.c_int, [_ctx_p, i64, C.c_double]),
            "pf_launch_count": (C.c_int, [_ctx_p, C.POINTER(i64)]),
            "pf_profile": (C.c_int, [_ctx_p, i32]),
            "pf_profile_read": (C.c_int, [_ctx_p, _D]),
            "pf_stream": (C.c_int, [_ctx_p, C.POINTER(C.c_void_p)]),
            "pf_debug_guards": (C.c_int, [_ctx_p, C.POINTER(i64), C.POINTER(i64)]),
            "pf_last_error": (C.c_char_p, [_ctx_p]),
            "pf_free": (None, [_ctx_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.pf_params_size() != C.sizeof(pf_params):
            raise ImportError(f"pf_params size mismatch: lib {L.pf_params_size()} vs binding {C.sizeof(pf_params)}")
        _lib = L
    return _lib


def _check(st, ctx=None):
    if st != PF_OK:
        msg = lib().pf_last_error(ctx)
        raise PfError(st, msg.decode() if msg else "")


def _dptr(a):
    if a is None:
        return None
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise TypeError("expected a C-contiguous float64 numpy array")
    return a.ctypes.data_as(_D)


def _hptr(a, need: int = 0):
    """Host pointer of a numpy array or of a pinned CPU torch tensor (float64, contiguous) holding at
    least `need` elements (the library writes / reads that many: a smaller buffer would be
    accessed out of bounds, so it is rejected here)."""
    if a is None:
        return None
    n = a.size if isinstance(a, np.ndarray) else (a.numel() if hasattr(a, "numel") else None)
    if need and n is not None and n < need:
        raise ValueError(f"host buffer holds {n} elements, the call needs {need}")
    if isinstance(a, np.ndarray):
        return _dptr(a)
    # torch tensor (pinned host memory for the e2e bench)
    if getattr(a, "device", None) is not None and str(a.device) != "cpu":
        raise TypeError("host buffers only")
    if str(a.dtype) != "torch.float64" or not a.is_contiguous():
        raise TypeError("expected a contiguous float64 tensor")
    return C.cast(C.c_void_p(a.data_ptr()), _D)


# ------------------------------------------------------------------ ABI-named functions
def pf_default_params(cfg: int) -> pf_params:
    p = pf_params()
    _check(lib().pf_default_params(cfg, C.byref(p)))
    return p


def pf_initial_fields(p: pf_params, member: int, y0: int, rows: int):
    c = np.empty((rows, p.nx)); phi = np.empty_like(c); rho = np.empty_like(c)
    _check(lib().pf_initial_fields(C.byref(p), member, y0, rows, _dptr(c), _dptr(phi), _dptr(rho)))
    return c, phi, rho


def pf_member_velocity(p: pf_params, member: int):
    vx, vy = C.c_double(), C.c_double()
    _check(lib().pf_member_velocity(C.byref(p), member, C.byref(vx), C.byref(vy)))
    return vx.value, vy.value


def pf_member_mobility(p: pf_params, member: int):
    """(M_A^bulk, M_B^bulk, M_A^surf, M_B^surf) of global member `member` (R-23)."""
    out = np.zeros(4)
    _check(lib().pf_member_mobility(C.byref(p), int(member), _dptr(out)))
    return tuple(float(x) for x in out)


def pf_inflow_row(p: pf_params, member: int, step: int) -> np.ndarray:
    out = np.zeros(p.nx)
    _check(lib().pf_inflow_row(C.byref(p), int(member), int(step), _dptr(out)))
    return out


def pf_dt_limit(p: pf_params) -> float:
    d = C.c_double()
    _check(lib().pf_dt_limit(C.byref(p), C.byref(d)))
    return d.value


def pf_create(p: pf_params):
    ctx = _ctx_p()
    _check(lib().pf_create(C.byref(p), C.byref(ctx)))
    return ctx


def pf_halo_plan(ny: int, nranks: int, rank: int):
    """(y0, ny_local, below, above, send_down_row, send_up_row, recv_below_row, recv_above_row)."""
    out = (C.c_int32 * 8)()
    _check(lib().pf_halo_plan(ny, nranks, rank, out))
    return tuple(out)


def pf_create_loopback(p: pf_params, nslabs: int):
    ctx = _ctx_p()
    _check(lib().pf_create_loopback(C.byref(p), nslabs, C.byref(ctx)))
    return ctx


def pf_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().pf_nccl_unique_id(buf))
    return buf.raw


def pf_create_slab(p: pf_params, rank: int, nranks: int, uid: bytes):
    if len(uid) != 128:
        raise ValueError("uid must be 128 bytes")
    ctx = _ctx_p()
    _check(lib().pf_create_slab(C.byref(p), rank, nranks, uid, C.byref(ctx)))
    return ctx


def pf_step(ctx, n: int):
    _check(lib().pf_step(ctx, int(n)), ctx)


def _field_elems(ctx, member):
    """Elements of one field buffer of pf_get/set_fields: local rows x nx (x members for -1)."""
    nx, _, mem = pf_shape(ctx)
    rows = pf_info(ctx)[3]
    return rows * nx * (mem if member == -1 else 1)


def pf_get_fields(ctx, member, c, phi, rho):
    n = _field_elems(ctx, member)
    _check(lib().pf_get_fields(ctx, member, _hptr(c, n), _hptr(phi, n), _hptr(rho, n)), ctx)


def pf_set_fields(ctx, member, c, phi, rho):
    n = _field_elems(ctx, member)
    _check(lib().pf_set_fields(ctx, member, _hptr(c, n), _hptr(phi, n), _hptr(rho, n)), ctx)


def pf_run_host(ctx, n, c_in, phi_in, rho_in, c_out, phi_out, rho_out, chunks: int = 4):
    k = _field_elems(ctx, -1)
    _check(lib().pf_run_host(ctx, int(n), _hptr(c_in, k), _hptr(phi_in, k), _hptr(rho_in, k), _hptr(c_out, k),
                             _hptr(phi_out, k), _hptr(rho_out, k), int(chunks)), ctx)


def pf_trajectory(ctx, n_snapshots: int, steps_between: int, out, times=None):
    """out: [members][n_snapshots][ny_local][nx] fp64 (numpy or pinned torch); times: [n_snapshots]."""
    k = _field_elems(ctx, -1) * int(n_snapshots)
    _check(lib().pf_trajectory(ctx, int(n_snapshots), int(steps_between), _hptr(out, k),
                               _hptr(times, int(n_snapshots))), ctx)


def pf_trajectory_file(ctx, path: str, n_snapshots: int, steps_between: int, dtype: str = "float64"):
    """Stream a trajectory to `path` (layout: include/pf.h pf_trajectory_file; read it back with
    read_trajectory)."""
    code = {"float64": 0, "float32": 1}[dtype]
    _check(lib().pf_trajectory_file(ctx, os.fsencode(path), n_snapshots, steps_between, code), ctx)


_TRAJ_HEADER = np.dtype([("magic", "S8"), ("header_bytes", "<u4"), ("version", "<u4"), ("nx", "<i4"),
                         ("ny_global", "<i4"), ("y0", "<i4"), ("ny_rows", "<i4"), ("members", "<i4"),
                         ("member_offset", "<i4"), ("n_snapshots", "<i4"), ("dtype", "<i4"),
                         ("steps_between", "<i8"), ("step0", "<i8"), ("dt", "<f8"), ("t0", "<f8"),
                         ("dx", "<f8"), ("rho_in", "<f8")])


def read_trajectory(path: str):
    """(header dict, member records [members, 8], snapshots as a read-only memmap [n_snapshots,
    members, ny_rows, nx], times [n_snapshots]) of a pf_trajectory_file file.  A dataset view
    [member][snapshot] is ``snaps.transpose(1, 0, 2, 3)``."""
    hdr = np.fromfile(path, dtype=_TRAJ_HEADER, count=1)[0]
    if hdr["magic"] != b"PFTRAJ01" or hdr["version"] != 1:
        raise ValueError(f"{path}: not a PFTRAJ01 v1 file")
    h = {k: (hdr[k].item() if k != "magic" else hdr[k].decode()) for k in _TRAJ_HEADER.names}
    M, S, ny, nx = h["members"], h["n_snapshots"], h["ny_rows"], h["nx"]
    recs = np.fromfile(path, dtype="<f8", count=8 * M, offset=_TRAJ_HEADER.itemsize).reshape(M, 8)
    dt = np.dtype("<f8") if h["dtype"] == 0 else np.dtype("<f4")
    snaps = np.memmap(path, dtype=dt, mode="r", offset=h["header_bytes"], shape=(S, M, ny, nx))
    times = np.fromfile(path, dtype="<f8", count=S, offset=h["header_bytes"] + S * M * ny * nx * dt.itemsize)
    if times.size != S:
        raise ValueError(f"{path}: truncated (no time footer)")
    return h, recs, snaps, times


def pf_s2(comp, threshold: float = 0.5, maps: bool = True, radial: bool = True):
    """S2 maps [batch][ny][nx] (centred) and radial profiles [batch][nbins] of composite fields
    comp [batch][ny][nx] (or [ny][nx]), computed on the GPU (NEXT-2)."""
    comp = np.ascontiguousarray(comp, dtype=np.float64)
    single = comp.ndim == 2
    if single:
        comp = comp[None]
    b, ny, nx = comp.shape
    nb = lib().pf_s2_nbins(nx, ny)
    s2 = np.empty_like(comp) if maps else None
    rad = np.empty((b, nb)) if radial else None
    _check(lib().pf_s2(_dptr(comp), nx, ny, b, float(threshold), _dptr(s2), _dptr(rad), nb))
    if single:
        s2 = None if s2 is None else s2[0]
        rad = None if rad is None else rad[0]
    return s2, rad


def pf_s2_rel_l2(comp_true, comp_pred, threshold: float = 0.5) -> np.ndarray:
    t = np.ascontiguousarray(comp_true, dtype=np.float64)
    p_ = np.ascontiguousarray(comp_pred, dtype=np.float64)
    if t.ndim == 2:
        t, p_ = t[None], p_[None]
    out = np.empty(t.shape[0])
    _check(lib().pf_s2_rel_l2(_dptr(t), _dptr(p_), t.shape[2], t.shape[1], t.shape[0], float(threshold), _dptr(out)))
    return out


def pf_diagnostics(ctx, member: int) -> np.ndarray:
    out = np.zeros(5)
    _check(lib().pf_diagnostics(ctx, member, _dptr(out)), ctx)
    return out


def pf_info(ctx):
    s, t, y0, ny = C.c_int64(), C.c_double(), C.c_int32(), C.c_int32()
    _check(lib().pf_info(ctx, C.byref(s), C.byref(t), C.byref(y0), C.byref(ny)), ctx)
    return s.value, t.value, y0.value, ny.value


def pf_shape(ctx):
    """(nx, ny, members) of the ctx."""
    nx, ny, m = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib().pf_shape(ctx, C.byref(nx), C.byref(ny), C.byref(m)), ctx)
    return nx.value, ny.value, m.value


def pf_set_time(ctx, steps: int, t: float):
    _check(lib().pf_set_time(ctx, steps, t), ctx)


def pf_launch_count(ctx) -> int:
    n = C.c_int64()
    _check(lib().pf_launch_count(ctx, C.byref(n)), ctx)
    return n.value


def pf_profile(ctx, enable: bool):
    _check(lib().pf_profile(ctx, 1 if enable else 0), ctx)


def pf_profile_read(ctx) -> np.ndarray:
    out = np.zeros(6)
    _check(lib().pf_profile_read(ctx, _dptr(out)), ctx)
    return out


def pf_stream(ctx) -> int:
    """cudaStream_t of the ctx as an integer handle (for torch.cuda.ExternalStream)."""
    s = C.c_void_p()
    _check(lib().pf_stream(ctx, C.byref(s)), ctx)
    return s.value or 0


def pf_debug_guards(ctx):
    """(guard bytes per zone, corrupted guard bytes) of a checked build (0, 0 in production)."""
    g, bad = C.c_int64(), C.c_int64()
    _check(lib().pf_debug_guards(ctx, C.byref(g), C.byref(bad)), ctx)
    return g.value, bad.value


def pf_free(ctx):
    if ctx:
        lib().pf_free(ctx)


# ------------------------------------------------------------------ convenience wrapper
class Simulation:
    """Owns one pf_ctx.  mode: 'single' | ('loopback', nslabs) | ('slab', rank, nranks, uid)."""

    def __init__(self, params: pf_params, mode="single"):
        self.params = params
        if mode == "single":
            self.ctx = pf_create(params)
        elif mode[0] == "loopback":
            self.ctx = pf_create_loopback(params, mode[1])
        elif mode[0] == "slab":
            self.ctx = pf_create_slab(params, mode[1], mode[2], mode[3])
        else:
            raise ValueError(mode)
        _, _, self.y0, self.ny_local = pf_info(self.ctx)

    @property
    def members(self):
        return self.params.n_members

    def step(self, n: int):
        pf_step(self.ctx, n)

    def fields(self, member: int = 0):
        shape = (self.ny_local, self.params.nx) if member >= 0 else (self.members, self.ny_local, self.params.nx)
        c = np.empty(shape); phi = np.empty(shape); rho = np.empty(shape)
        pf_get_fields(self.ctx, member, c, phi, rho)
        return c, phi, rho

    def set_fields(self, member, c=None, phi=None, rho=None):
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        pf_set_fields(self.ctx, member, f(c), f(phi), f(rho))

    def diagnostics(self, member: int = 0):
        return pf_diagnostics(self.ctx, member)

    def info(self):
        return pf_info(self.ctx)

    def close(self):
        if self.ctx:
            pf_free(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
