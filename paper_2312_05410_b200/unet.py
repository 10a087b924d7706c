"""Thin ctypes binding of the U-Net inference ABI (include/unet.h, NEXT-4): argument marshalling only.

Every step of the forward pass runs in libpf.so's kernels (tcgen05 implicit-GEMM convolutions,
GroupNorm / GELU / conditioning / pooling / up-sampling kernels, the time MLP).  There is no CPU
fallback: without the library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import pf

UN_ABI_VERSION = 1


class un_params(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("lb", C.c_int32), ("widths", C.c_int32 * 4),
                ("height", C.c_int32), ("width", C.c_int32), ("max_batch", C.c_int32), ("device", C.c_int32)]


_ready = False
_F = C.POINTER(C.c_float)


def lib():
    global _ready
    L = pf.lib()
    if not _ready:
        P = C.POINTER(un_params)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "un_default_params": (C.c_int, [P]),
            "un_blob_size": (i64, [P]),
            "un_create": (C.c_int, [P, C.POINTER(vp)]),
            "un_set_weights": (C.c_int, [vp, _F, i64]),
            "un_forward_device": (C.c_int, [vp, i32, vp, vp, vp]),
            "un_forward": (C.c_int, [vp, i32, _F, _F, _F]),
            "un_rollout": (C.c_int, [vp, i32, _F, i32, i32, _F]),
            "un_conv3x3": (C.c_int, [vp, i32, i32, i32, i32, vp, i32, vp, vp]),
            "un_hybrid": (C.c_int, [vp, vp, i32, i64, i32, i32, _F, C.POINTER(C.c_double)]),
            "un_stream": (C.c_int, [vp, C.POINTER(vp)]),
            "un_launch_count": (C.c_int, [vp, C.POINTER(i64)]),
            "un_profile": (C.c_int, [vp, i32]),
            "un_profile_read": (C.c_int, [vp, C.POINTER(C.c_double)]),
            "un_last_error": (C.c_char_p, [vp]),
            "un_free": (None, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _ready = True
    return L


def _check(st, ctx=None):
    if st != 0:
        msg = lib().un_last_error(ctx)
        raise pf.PfError(st, msg.decode() if msg else "")


def default_params(**kw):
    p = un_params()
    _check(lib().un_default_params(C.byref(p)))
    for k, v in kw.items():
        if k == "widths":
            p.widths = (C.c_int32 * 4)(*v)
        else:
            setattr(p, k, v)
    return p


def blob_size(p):
    return int(lib().un_blob_size(C.byref(p)))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def conv3x3(inp, w, out, batch, H, W, cin, cout, stream=0):
    """Device pointers (ints): inp bf16 [batch*H*W][cin], w bf16 [cout][9][cin], out fp32."""
    _check(lib().un_conv3x3(C.c_void_p(inp), batch, H, W, cin, C.c_void_p(w), cout, C.c_void_p(out),
                            C.c_void_p(stream)))


class UNet:
    """Owns an un_ctx: weights, activations and a stream on the device."""

    def __init__(self, params=None, weights=None):
        self.p = params if params is not None else default_params()
        h = C.c_void_p()
        _check(lib().un_create(C.byref(self.p), C.byref(h)))
        self.ctx = h
        if weights is not None:
            self.set_weights(weights)

    def set_weights(self, blob):
        b = _f32(blob)
        _check(lib().un_set_weights(self.ctx, b.ctypes.data_as(_F), b.size), self.ctx)

    def _check_hist(self, hist):
        """The library copies B * lb * H * W floats from the pointer: a wrongly shaped array would be
        read out of bounds, so the shape is checked here."""
        want = (self.p.lb, self.p.height, self.p.width)
        if np.ndim(hist) != 4 or tuple(np.shape(hist)[1:]) != want:
            raise ValueError(f"hist must have shape (B, {want[0]}, {want[1]}, {want[2]}), got {np.shape(hist)}")
        if not 1 <= np.shape(hist)[0] <= self.p.max_batch:
            raise ValueError(f"batch {np.shape(hist)[0]} outside [1, max_batch = {self.p.max_batch}]")

    def forward(self, hist, dt, out=None):
        """hist [B, lb, H, W], dt [B] or scalar (host) -> [B, H, W] float32 (host; written into `out`
        when given, e.g. a page-locked array, which lets un_forward overlap its copies)."""
        self._check_hist(hist)
        if np.ndim(dt) not in (0, 1) or (np.ndim(dt) == 1 and np.shape(dt)[0] != np.shape(hist)[0]):
            raise ValueError(f"dt must be a scalar or have shape ({np.shape(hist)[0]},), got {np.shape(dt)}")
        h, d = _f32(hist), _f32(np.broadcast_to(dt, (hist.shape[0],)))
        shape = (h.shape[0], self.p.height, self.p.width)
        if out is None:
            out = np.empty(shape, dtype=np.float32)
        elif out.shape != shape or out.dtype != np.float32 or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a C-contiguous float32 array of shape {shape}")
        _check(lib().un_forward(self.ctx, h.shape[0], h.ctypes.data_as(_F), d.ctypes.data_as(_F),
                                out.ctypes.data_as(_F)), self.ctx)
        return out

    def forward_device(self, batch, hist_ptr, dt_ptr, out_ptr):
        _check(lib().un_forward_device(self.ctx, batch, C.c_void_p(hist_ptr), C.c_void_p(dt_ptr),
                                       C.c_void_p(out_ptr)), self.ctx)

    def rollout(self, hist, lf, n_leaps):
        self._check_hist(hist)
        h = _f32(hist)
        out = np.empty((h.shape[0], n_leaps * lf, self.p.height, self.p.width), dtype=np.float32)
        _check(lib().un_rollout(self.ctx, h.shape[0], h.ctypes.data_as(_F), lf, n_leaps,
                                out.ctypes.data_as(_F)), self.ctx)
        return out

    def hybrid(self, sim, n_dns, steps_between, lf, n_leaps):
        """DNS (pf ctx of `sim`) for n_dns composite snapshots, then the U-Net rollout; returns
        (snapshots [members, n_dns + n_leaps*lf, H, W], (dns_seconds, surrogate_seconds))."""
        nx, ny, mem = pf.pf_shape(sim.ctx)
        shape = (mem, n_dns + n_leaps * lf, ny, nx)
        try:   # pinned host memory: the predictions are copied asynchronously at full PCIe rate
            import torch
            self._pinned = torch.empty(shape, dtype=torch.float32, pin_memory=True)
            out = self._pinned.numpy()
        except Exception:
            out = np.zeros(shape, dtype=np.float32)   # pre-faulted pageable pages
        sec = (C.c_double * 2)()
        _check(lib().un_hybrid(self.ctx, sim.ctx, n_dns, steps_between, lf, n_leaps, out.ctypes.data_as(_F), sec),
               self.ctx)
        return out, (sec[0], sec[1])

    def stream(self):
        s = C.c_void_p()
        _check(lib().un_stream(self.ctx, C.byref(s)), self.ctx)
        return s.value or 0

    def launches(self):
        n = C.c_int64()
        _check(lib().un_launch_count(self.ctx, C.byref(n)), self.ctx)
        return n.value

    def profile(self, enable):
        _check(lib().un_profile(self.ctx, int(enable)), self.ctx)

    def profile_read(self):
        out = (C.c_double * 4)()
        _check(lib().un_profile_read(self.ctx, out), self.ctx)
        return list(out)

    def close(self):
        if self.ctx:
            lib().un_free(self.ctx)
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
