"""Thin ctypes binding of libifdk (include/ifdk.h): argument marshalling only.

Every step of the FDK hot path runs in the CUDA kernels of libifdk.so; this
module only converts torch tensors / numpy arrays into pointers and sizes and
turns non-OK statuses into exceptions.  There is no CPU fallback: if the
library is missing the import fails, and without a GPU every compute call
raises ``IfdkError`` (status IFDK_ERR_CUDA).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libifdk.so")

IFDK_OK = 0
STATUS_NAMES = {
    0: "IFDK_OK",
    1: "IFDK_ERR_INVALID_ARGUMENT",
    2: "IFDK_ERR_DEGENERATE_GEOMETRY",
    3: "IFDK_ERR_SHAPE",
    4: "IFDK_ERR_CUDA",
    5: "IFDK_ERR_OUT_OF_MEMORY",
}

# Every symbol include/ifdk.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ifdk_geometry_create",
    "ifdk_geometry_destroy",
    "ifdk_projection_matrix",
    "ifdk_band_rows",
    "ifdk_filter",
    "ifdk_filter_scatter",
    "ifdk_peer_alloc",
    "ifdk_peer_open",
    "ifdk_peer_close",
    "ifdk_peer_free",
    "ifdk_signal",
    "ifdk_wait",
    "ifdk_backproject_reduce",
    "ifdk_backproject",
    "ifdk_backproject_alg2",
    "ifdk_backproject_alg4",
    "ifdk_reconstruct",
    "ifdk_reconstruct_host",
    "ifdk_reconstruct_slab_host",
    "ifdk_forward_project",
    "ifdk_sart_ratio",
    "ifdk_sart_update",
    "ifdk_mlem_ratio",
    "ifdk_mlem_update",
    "ifdk_fill",
    "ifdk_set_bp_variant",
    "ifdk_last_launch_count",
    "ifdk_last_error",
)


class IfdkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing -- build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the iFDK path has no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)
_vp, _i, _l, _d = ctypes.c_void_p, ctypes.c_int, ctypes.c_long, ctypes.c_double
_lib.ifdk_geometry_create.argtypes = [_i] * 5 + [_d] * 8 + [ctypes.POINTER(_vp)]
_lib.ifdk_geometry_create.restype = _i
_lib.ifdk_geometry_destroy.argtypes = [_vp]
_lib.ifdk_geometry_destroy.restype = None
_lib.ifdk_projection_matrix.argtypes = [_vp, _l, ctypes.POINTER(_d)]
_lib.ifdk_projection_matrix.restype = _i
_lib.ifdk_band_rows.argtypes = [_vp, _i, _i, _l, ctypes.POINTER(_i), ctypes.POINTER(_i)]
_lib.ifdk_band_rows.restype = _i
_lib.ifdk_filter.argtypes = [_vp, _vp, _vp, _l, _i, _i, _vp]
_lib.ifdk_filter.restype = _i
class _BandDest(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("v_lo", ctypes.c_int), ("v_hi", ctypes.c_int)]


_lib.ifdk_filter_scatter.argtypes = [_vp, _vp, _l, _i, _i, _i, ctypes.POINTER(_BandDest), _i,
                                     ctypes.POINTER(_vp), _vp, _vp]
_lib.ifdk_filter_scatter.restype = _i
_lib.ifdk_peer_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(_vp), ctypes.c_char_p]
_lib.ifdk_peer_alloc.restype = _i
_lib.ifdk_peer_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(_vp)]
_lib.ifdk_peer_open.restype = _i
_lib.ifdk_peer_close.argtypes = [_vp]
_lib.ifdk_peer_close.restype = _i
_lib.ifdk_peer_free.argtypes = [_vp]
_lib.ifdk_peer_free.restype = _i
_lib.ifdk_signal.argtypes = [_i, ctypes.POINTER(_vp), _vp]
_lib.ifdk_signal.restype = _i
_lib.ifdk_wait.argtypes = [_vp, _i, ctypes.c_uint, ctypes.c_uint, _vp]
_lib.ifdk_wait.restype = _i
_lib.ifdk_backproject.argtypes = [_vp, _vp, _l, _l, _i, _i, _vp, _i, _i, _i, _vp]
_lib.ifdk_backproject.restype = _i
_lib.ifdk_backproject_reduce.argtypes = [_vp, _vp, _l, _l, _i, _i, _i, _i, _i,
                                         ctypes.POINTER(_vp), ctypes.POINTER(_i), _i, _vp]
_lib.ifdk_backproject_reduce.restype = _i
_lib.ifdk_backproject_alg2.argtypes = [_vp, _vp, _l, _l, _vp, _i, _i, _i, _i, _vp]
_lib.ifdk_backproject_alg2.restype = _i
_lib.ifdk_backproject_alg4.argtypes = [_vp, _vp, _l, _l, _vp, _i, _i, _vp]
_lib.ifdk_backproject_alg4.restype = _i
_lib.ifdk_reconstruct.argtypes = [_vp, _vp, _l, _vp, _vp]
_lib.ifdk_reconstruct.restype = _i
_lib.ifdk_reconstruct_host.argtypes = [_vp, _vp, _l, _vp, _vp]
_lib.ifdk_reconstruct_host.restype = _i
_lib.ifdk_reconstruct_slab_host.argtypes = [_vp, _vp, _l, _i, _i, _vp, _vp]
_lib.ifdk_reconstruct_slab_host.restype = _i
_lib.ifdk_forward_project.argtypes = [_vp, _vp, _i, _i, _l, _l, _vp, _i, _i, _i, _vp]
_lib.ifdk_forward_project.restype = _i
_lib.ifdk_sart_ratio.argtypes = [_vp, _vp, _vp, _vp, _l, _vp]
_lib.ifdk_sart_ratio.restype = _i
_lib.ifdk_sart_update.argtypes = [_vp, _vp, _vp, ctypes.c_float, _l, _i, _vp]
_lib.ifdk_sart_update.restype = _i
_lib.ifdk_mlem_ratio.argtypes = [_vp, _vp, _vp, _l, _vp]
_lib.ifdk_mlem_ratio.restype = _i
_lib.ifdk_mlem_update.argtypes = [_vp, _vp, _vp, _l, _vp]
_lib.ifdk_mlem_update.restype = _i
_lib.ifdk_fill.argtypes = [_vp, ctypes.c_float, _l, _vp]
_lib.ifdk_fill.restype = _i
_lib.ifdk_set_bp_variant.argtypes = [_i, _i]
_lib.ifdk_set_bp_variant.restype = _i
_lib.ifdk_last_launch_count.argtypes = []
_lib.ifdk_last_launch_count.restype = _i
_lib.ifdk_last_error.argtypes = []
_lib.ifdk_last_error.restype = ctypes.c_char_p


def _check(st: int) -> None:
    if st != IFDK_OK:
        raise IfdkError(st, _lib.ifdk_last_error().decode())


def set_bp_variant(walk: int = 0, raster: int = 0) -> None:
    """Speed-tuning hook (A/B runs, tests): pick a back-projection walk (include/ifdk.h lists
    the families; variants within a family are bitwise equal) and the CTA raster band;
    0 = automatic."""
    _check(_lib.ifdk_set_bp_variant(int(walk), int(raster)))


def last_launch_count() -> int:
    """Kernels the last successful libifdk call on this thread launched."""
    return int(_lib.ifdk_last_launch_count())


class Geometry:
    """ifdk_geometry_create / ifdk_geometry_destroy (Table tbl:cbct-param)."""

    def __init__(self, Nu, Nv, Nx, Ny, Nz, Du, Dv, Dx, Dy, Dz, D, d, theta):
        h = _vp()
        _check(_lib.ifdk_geometry_create(int(Nu), int(Nv), int(Nx), int(Ny), int(Nz), float(Du),
                                         float(Dv), float(Dx), float(Dy), float(Dz), float(D),
                                         float(d), float(theta), ctypes.byref(h)))
        self._h = h
        self.Nu, self.Nv, self.Nx, self.Ny, self.Nz = int(Nu), int(Nv), int(Nx), int(Ny), int(Nz)
        self.Du, self.Dv, self.Dx, self.Dy, self.Dz = map(float, (Du, Dv, Dx, Dy, Dz))
        self.D, self.d, self.theta = float(D), float(d), float(theta)

    @classmethod
    def from_spec(cls, spec) -> "Geometry":
        return cls(**spec.geometry_args())

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.ifdk_geometry_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def projection_matrix(self, s: int) -> np.ndarray:
        P = (ctypes.c_double * 12)()
        _check(_lib.ifdk_projection_matrix(self._h, int(s), P))
        return np.frombuffer(P, np.float64).reshape(3, 4).copy()

    def band_rows(self, k0: int, nk: int, s: int) -> tuple[int, int]:
        lo, hi = ctypes.c_int(), ctypes.c_int()
        _check(_lib.ifdk_band_rows(self._h, int(k0), int(nk), int(s), ctypes.byref(lo),
                                   ctypes.byref(hi)))
        return lo.value, hi.value


def _stream_ptr(stream) -> int:
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _dev_f32(t, name):
    import torch

    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda:
        raise TypeError(f"{name} must be a float32 CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def ifdk_filter(g: Geometry, raw, filtered, v0: int = 0, stream=None) -> None:
    """filtered = Alg. alg:filter(raw) for rows v0.. of each view; tensors [n_views][n_rows][Nu]."""
    if tuple(raw.shape) != tuple(filtered.shape) or raw.dim() != 3 or raw.shape[2] != g.Nu:
        raise ValueError("raw and filtered must both be [n_views][n_rows][Nu]")
    _check(_lib.ifdk_filter(g.handle, _dev_f32(raw, "raw"), _dev_f32(filtered, "filtered"),
                            raw.shape[0], int(v0), raw.shape[1], _stream_ptr(stream)))


def _ptr_array(ptrs):
    return (_vp * max(len(ptrs), 1))(*[int(x) for x in ptrs])


def ifdk_filter_scatter(g: Geometry, raw, dests, v0: int = 0, flags=(), ticket: int = 0,
                        stream=None) -> None:
    """Alg. alg:filter of raw [n_views][n_rows][Nu] (rows v0..), each filtered row stored into
    every destination band that holds it.  dests: list of (ptr, v_lo, v_hi) where ptr is a
    device pointer (int: tensor.data_ptr() or a peer-mapped ifdk_peer_open address) to an
    [n_views][v_hi - v_lo + 1][Nu] fp32 buffer.  flags: device pointers of uint32 words, each
    incremented once all rows have landed (system scope); ticket: a device uint32 word that is
    0 (required with flags)."""
    if raw.dim() != 3 or raw.shape[2] != g.Nu:
        raise ValueError("raw must be [n_views][n_rows][Nu]")
    arr = (_BandDest * len(dests))(*[_BandDest(int(b), int(lo), int(hi)) for b, lo, hi in dests])
    _check(_lib.ifdk_filter_scatter(g.handle, _dev_f32(raw, "raw"), raw.shape[0], int(v0),
                                    raw.shape[1], len(dests), arr, len(flags), _ptr_array(flags),
                                    int(ticket) or None, _stream_ptr(stream)))


def peer_alloc(nbytes: int) -> tuple[int, bytes]:
    """ifdk_peer_alloc: (device pointer, 64-byte IPC handle) of a fresh cudaMalloc."""
    ptr = _vp()
    h = ctypes.create_string_buffer(64)
    _check(_lib.ifdk_peer_alloc(int(nbytes), ctypes.byref(ptr), h))
    return int(ptr.value), bytes(h.raw)


def peer_open(handle: bytes) -> int:
    """ifdk_peer_open: map another process's peer buffer; returns its device pointer here."""
    ptr = _vp()
    _check(_lib.ifdk_peer_open(bytes(handle), ctypes.byref(ptr)))
    return int(ptr.value)


def peer_close(ptr: int) -> None:
    _check(_lib.ifdk_peer_close(int(ptr) or None))


def peer_free(ptr: int) -> None:
    _check(_lib.ifdk_peer_free(int(ptr) or None))


def ifdk_signal(flags, stream=None) -> None:
    """After earlier work on the stream, each device uint32 word in `flags` += 1 (system scope)."""
    _check(_lib.ifdk_signal(len(flags), _ptr_array(flags), _stream_ptr(stream)))


def ifdk_wait(flags_ptr: int, n: int, target: int, timeout_ms: int = 0, stream=None) -> None:
    """Later work on the stream waits until the n uint32 words at flags_ptr reach target
    (a trap after timeout_ms, 0 = 300 s)."""
    _check(_lib.ifdk_wait(int(flags_ptr), int(n), int(target) & 0xFFFFFFFF, int(timeout_ms),
                          _stream_ptr(stream)))


class DeviceArray:
    """A CUDA array view of raw device memory (e.g. a peer buffer) for torch.as_tensor:
    __cuda_array_interface__ with the caller keeping the memory alive."""

    def __init__(self, ptr: int, shape, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}


def as_tensor(ptr: int, shape, dtype: str = "float32"):
    """torch tensor over device memory at ptr (no copy; memory owned elsewhere)."""
    import torch

    ts = {"float32": "<f4", "uint32": "<u4", "int32": "<i4"}[dtype]
    return torch.as_tensor(DeviceArray(ptr, shape, ts), device="cuda")


def ifdk_backproject(g: Geometry, filtered, s0: int, vol, k0: int = 0, v0: int = 0,
                     accumulate: bool = False, stream=None) -> None:
    """vol (=|+=) Alg. alg:bp over views s0..s0+n-1; filtered [n][n_rows][Nu] holds rows v0..,
    vol [nk][Ny][Nx] is the slab k0..k0+nk-1."""
    if filtered.dim() != 3 or filtered.shape[2] != g.Nu:
        raise ValueError("filtered must be [n_views][n_rows][Nu]")
    if vol.dim() != 3 or vol.shape[1] != g.Ny or vol.shape[2] != g.Nx:
        raise ValueError("vol must be [nk][Ny][Nx]")
    _check(_lib.ifdk_backproject(g.handle, _dev_f32(filtered, "filtered"), int(s0),
                                 filtered.shape[0], int(v0), filtered.shape[1],
                                 _dev_f32(vol, "vol"), int(k0), vol.shape[0],
                                 1 if accumulate else 0, _stream_ptr(stream)))


def ifdk_backproject_reduce(g: Geometry, filtered, s0: int, dests, dest_k0, k0: int = 0,
                            nk: int | None = None, v0: int = 0, mode: int = 0,
                            stream=None) -> None:
    """Fused projection-split BP: views s0.. (filtered [n][n_rows][Nu], rows v0..) over slices
    k0..k0+nk-1, each 128-view partial sum ADDED (red.global.add, mode 0; multimem.red, mode
    1) into the destination slab holding its slice: dests[d] (device pointers or tensors,
    local or peer-mapped) holds slices dest_k0[d] .. dest_k0[d+1]-1."""
    if filtered.dim() != 3 or filtered.shape[2] != g.Nu:
        raise ValueError("filtered must be [n_views][n_rows][Nu]")
    nk = g.Nz - k0 if nk is None else nk
    ptrs = [d if isinstance(d, int) else _dev_f32(d, "dest") for d in dests]
    if len(ptrs) != len(dest_k0):
        raise ValueError("one start slice per destination slab")
    arr = (_vp * len(ptrs))(*ptrs)
    ks = (_i * len(dest_k0))(*[int(k) for k in dest_k0])
    _check(_lib.ifdk_backproject_reduce(g.handle, _dev_f32(filtered, "filtered"), int(s0),
                                        filtered.shape[0], int(v0), filtered.shape[1], int(k0),
                                        int(nk), len(ptrs), arr, ks, int(mode),
                                        _stream_ptr(stream)))


def ifdk_backproject_alg2(g: Geometry, filtered, s0: int, vol, k0: int = 0,
                          accumulate: bool = False, texture: bool = True, stream=None) -> None:
    """MEASURED BASELINE (not the production path): the paper's per-voxel fp32 Alg. alg:bp with
    hardware-texture (texture=True) or software bilinear sampling; filtered [n][Nv][Nu]."""
    if filtered.dim() != 3 or filtered.shape[1] != g.Nv or filtered.shape[2] != g.Nu:
        raise ValueError("filtered must be [n_views][Nv][Nu]")
    if vol.dim() != 3 or vol.shape[1] != g.Ny or vol.shape[2] != g.Nx:
        raise ValueError("vol must be [nk][Ny][Nx]")
    _check(_lib.ifdk_backproject_alg2(g.handle, _dev_f32(filtered, "filtered"), int(s0),
                                      filtered.shape[0], _dev_f32(vol, "vol"), int(k0),
                                      vol.shape[0], 1 if accumulate else 0, 1 if texture else 0,
                                      _stream_ptr(stream)))


def ifdk_backproject_alg4(g: Geometry, filtered, s0: int, vol, accumulate: bool = False,
                          texture: bool = False, stream=None) -> None:
    """MEASURED BASELINE: the paper's Alg. alg:bp-v1 (fp32, mirror k-pairs) over the whole
    volume; filtered [n][Nv][Nu], vol [Nz][Ny][Nx]."""
    if filtered.dim() != 3 or filtered.shape[1] != g.Nv or filtered.shape[2] != g.Nu:
        raise ValueError("filtered must be [n_views][Nv][Nu]")
    if tuple(vol.shape) != (g.Nz, g.Ny, g.Nx):
        raise ValueError("vol must be [Nz][Ny][Nx]")
    _check(_lib.ifdk_backproject_alg4(g.handle, _dev_f32(filtered, "filtered"), int(s0),
                                      filtered.shape[0], _dev_f32(vol, "vol"),
                                      1 if accumulate else 0, 1 if texture else 0,
                                      _stream_ptr(stream)))


def ifdk_reconstruct(g: Geometry, raw, vol, stream=None) -> None:
    """vol = FDK(raw): raw [n_views][Nv][Nu] device, vol [Nz][Ny][Nx] device."""
    if raw.dim() != 3 or raw.shape[1] != g.Nv or raw.shape[2] != g.Nu:
        raise ValueError("raw must be [n_views][Nv][Nu]")
    if tuple(vol.shape) != (g.Nz, g.Ny, g.Nx):
        raise ValueError("vol must be [Nz][Ny][Nx]")
    _check(_lib.ifdk_reconstruct(g.handle, _dev_f32(raw, "raw"), raw.shape[0],
                                 _dev_f32(vol, "vol"), _stream_ptr(stream)))


def _host_f32(a, name):
    import torch

    if isinstance(a, torch.Tensor):
        if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous():
            raise TypeError(f"{name} must be a contiguous float32 host tensor")
        return a.data_ptr(), tuple(a.shape)
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags.c_contiguous:
        raise TypeError(f"{name} must be a C-contiguous float32 array")
    return a.ctypes.data, a.shape


def ifdk_reconstruct_host(g: Geometry, raw_host, vol_host, stream=None) -> None:
    """End-to-end FDK from host memory (H2D, filter, back-project, D2H); synchronous."""
    rp, rs = _host_f32(raw_host, "raw_host")
    vp, vs = _host_f32(vol_host, "vol_host")
    if len(rs) != 3 or rs[1] != g.Nv or rs[2] != g.Nu:
        raise ValueError("raw_host must be [n_views][Nv][Nu]")
    if tuple(vs) != (g.Nz, g.Ny, g.Nx):
        raise ValueError("vol_host must be [Nz][Ny][Nx]")
    _check(_lib.ifdk_reconstruct_host(g.handle, rp, rs[0], vp, _stream_ptr(stream)))


def ifdk_reconstruct_slab_host(g: Geometry, raw_host, k0: int, vol_host, stream=None) -> None:
    """Slab k0..k0+nk-1 (vol_host [nk][Ny][Nx], host) reconstructed from host views
    raw_host [n][Nv][Nu] copying only the slab's detector row band (no exchange); synchronous."""
    rp, rs = _host_f32(raw_host, "raw_host")
    vp, vs = _host_f32(vol_host, "vol_host")
    if len(rs) != 3 or rs[1] != g.Nv or rs[2] != g.Nu:
        raise ValueError("raw_host must be [n_views][Nv][Nu]")
    if len(vs) != 3 or vs[1] != g.Ny or vs[2] != g.Nx:
        raise ValueError("vol_host must be [nk][Ny][Nx]")
    _check(_lib.ifdk_reconstruct_slab_host(g.handle, rp, rs[0], int(k0), vs[0], vp,
                                           _stream_ptr(stream)))


def ifdk_forward_project(g: Geometry, vol, s0: int, proj, k0: int = 0, v0: int = 0,
                         accumulate: bool = False, stream=None) -> None:
    """proj (=|+=) the matched forward projection (transpose of ifdk_backproject) of the slab
    vol [nk][Ny][Nx] (k0..) for views s0..s0+n-1; proj [n][n_rows][Nu] holds rows v0.."""
    if proj.dim() != 3 or proj.shape[2] != g.Nu:
        raise ValueError("proj must be [n_views][n_rows][Nu]")
    if vol.dim() != 3 or vol.shape[1] != g.Ny or vol.shape[2] != g.Nx:
        raise ValueError("vol must be [nk][Ny][Nx]")
    _check(_lib.ifdk_forward_project(g.handle, _dev_f32(vol, "vol"), int(k0), vol.shape[0],
                                     int(s0), proj.shape[0], _dev_f32(proj, "proj"), int(v0),
                                     proj.shape[1], 1 if accumulate else 0, _stream_ptr(stream)))


def ifdk_sart_ratio(b, ax, R, out, stream=None) -> None:
    """out = (b - ax) / R (0 where R <= 0); equal-size float32 CUDA tensors."""
    n = b.numel()
    if not (ax.numel() == R.numel() == out.numel() == n):
        raise ValueError("b, ax, R and out must have the same size")
    _check(_lib.ifdk_sart_ratio(_dev_f32(b, "b"), _dev_f32(ax, "ax"), _dev_f32(R, "R"),
                                _dev_f32(out, "out"), n, _stream_ptr(stream)))


def ifdk_sart_update(x, c, C, lam: float, nonneg: bool = False, stream=None) -> None:
    """x += lam c / C (unchanged where C <= 0), optionally clamped at 0."""
    n = x.numel()
    if not (c.numel() == C.numel() == n):
        raise ValueError("x, c and C must have the same size")
    _check(_lib.ifdk_sart_update(_dev_f32(x, "x"), _dev_f32(c, "c"), _dev_f32(C, "C"),
                                 float(lam), n, 1 if nonneg else 0, _stream_ptr(stream)))


def ifdk_mlem_ratio(b, ax, out, stream=None) -> None:
    """out = b / ax where ax > 0, else 0; equal-size float32 CUDA tensors."""
    n = b.numel()
    if not (ax.numel() == out.numel() == n):
        raise ValueError("b, ax and out must have the same size")
    _check(_lib.ifdk_mlem_ratio(_dev_f32(b, "b"), _dev_f32(ax, "ax"), _dev_f32(out, "out"), n,
                                _stream_ptr(stream)))


def ifdk_mlem_update(x, c, C, stream=None) -> None:
    """x = x c / C where C > 0 (else unchanged)."""
    n = x.numel()
    if not (c.numel() == C.numel() == n):
        raise ValueError("x, c and C must have the same size")
    _check(_lib.ifdk_mlem_update(_dev_f32(x, "x"), _dev_f32(c, "c"), _dev_f32(C, "C"), n,
                                 _stream_ptr(stream)))


def ifdk_fill(x, value: float, stream=None) -> None:
    """x[:] = value on the device."""
    _check(_lib.ifdk_fill(_dev_f32(x, "x"), float(value), x.numel(), _stream_ptr(stream)))
