"""ctypes front end of oracle.c plus the fp64 FFT form of the filter.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2, OpenMP, no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99", _SRC, "-o", _LIB, "-lm"]
        )
    return _LIB


class _CGeom(ctypes.Structure):
    _fields_ = [
        ("Nu", ctypes.c_int), ("Nv", ctypes.c_int),
        ("Nx", ctypes.c_int), ("Ny", ctypes.c_int), ("Nz", ctypes.c_int),
        ("Du", ctypes.c_double), ("Dv", ctypes.c_double),
        ("Dx", ctypes.c_double), ("Dy", ctypes.c_double), ("Dz", ctypes.c_double),
        ("D", ctypes.c_double), ("d", ctypes.c_double), ("theta", ctypes.c_double),
    ]


@dataclass(frozen=True)
class OracleGeometry:
    """Table tbl:cbct-param.  theta is the angle step; beta_s = s*theta."""

    Nu: int
    Nv: int
    Nx: int
    Ny: int
    Nz: int
    Du: float
    Dv: float
    Dx: float
    Dy: float
    Dz: float
    D: float
    d: float
    theta: float

    def c(self) -> _CGeom:
        return _CGeom(self.Nu, self.Nv, self.Nx, self.Ny, self.Nz, self.Du, self.Dv,
                      self.Dx, self.Dy, self.Dz, self.D, self.d, self.theta)


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        ip = ctypes.POINTER(ctypes.c_int)
        g = ctypes.POINTER(_CGeom)
        _lib.oracle_projection_matrix.argtypes = [g, ctypes.c_long, dp]
        _lib.oracle_cos_weight.argtypes = [g, ctypes.c_int, ctypes.c_int]
        _lib.oracle_cos_weight.restype = ctypes.c_double
        _lib.oracle_ramp_h1.argtypes = [ctypes.c_long]
        _lib.oracle_ramp_h1.restype = ctypes.c_double
        _lib.oracle_fdk_scale.argtypes = [g]
        _lib.oracle_fdk_scale.restype = ctypes.c_double
        _lib.oracle_filter.argtypes = [g, fp, ctypes.c_long, ctypes.c_int, ctypes.c_int, dp]
        _lib.oracle_interp2.argtypes = [g, dp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ip]
        _lib.oracle_interp2.restype = ctypes.c_double
        _lib.oracle_backproject.argtypes = [g, dp, ctypes.c_long, ctypes.c_long, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_long, ip, dp]
        _lib.oracle_backproject.restype = ctypes.c_int
        _lib.oracle_backproject_volume.argtypes = [g, dp, ctypes.c_long, ctypes.c_long,
                                                   ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int, dp]
        _lib.oracle_backproject_volume.restype = ctypes.c_int
        _lib.oracle_forward_project.argtypes = [g, dp, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                                ctypes.c_long, ctypes.c_int, ctypes.c_int, dp]
        _lib.oracle_forward_project.restype = ctypes.c_int
        _lib.oracle_num_threads.restype = ctypes.c_int
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def num_threads() -> int:
    return int(_L().oracle_num_threads())


def projection_matrix(g: OracleGeometry, s: int) -> np.ndarray:
    """P_s (3x4, fp64) as the product of the printed matrices."""
    P = np.zeros(12, np.float64)
    cg = g.c()
    _L().oracle_projection_matrix(ctypes.byref(cg), int(s), _ptr(P, ctypes.c_double))
    return P.reshape(3, 4)


def cos_weight(g: OracleGeometry, m: int, v: int) -> float:
    cg = g.c()
    return float(_L().oracle_cos_weight(ctypes.byref(cg), int(m), int(v)))


def ramp_h1(n: int) -> float:
    return float(_L().oracle_ramp_h1(int(n)))


def fdk_scale(g: OracleGeometry) -> float:
    cg = g.c()
    return float(_L().oracle_fdk_scale(ctypes.byref(cg)))


def filter_direct(g: OracleGeometry, E: np.ndarray, v0: int = 0) -> np.ndarray:
    """Alg. alg:filter, direct sum.  E: [n_views][n_rows][Nu] fp32 holding rows v0.. ."""
    E = np.ascontiguousarray(E, dtype=np.float32)
    assert E.ndim == 3 and E.shape[2] == g.Nu
    Q = np.empty(E.shape, np.float64)
    cg = g.c()
    _L().oracle_filter(ctypes.byref(cg), _ptr(E, ctypes.c_float), E.shape[0], int(v0),
                       E.shape[1], _ptr(Q, ctypes.c_double))
    return Q


def filter_fft(g: OracleGeometry, E: np.ndarray, v0: int = 0, workers: int = -1) -> np.ndarray:
    """Alg. alg:filter with the convolution done by the convolution theorem
    (P:448-454): zero-pad each cosine-weighted row to L >= 2 Nu - 1, multiply
    by the DFT of h1 laid out circularly for lags -(Nu-1)..(Nu-1), invert,
    keep samples 0..Nu-1.  Library fp64 FFT (scipy.fft)."""
    import scipy.fft as sfft

    E = np.asarray(E)
    n_views, n_rows, Nu = E.shape
    assert Nu == g.Nu
    L = 1
    while L < 2 * Nu - 1:
        L *= 2
    lags = np.arange(L)
    lags = np.where(lags < L // 2 + 1, lags, lags - L)  # circular lag of each slot
    h = np.array([ramp_h1(int(n)) if abs(n) <= Nu - 1 else 0.0 for n in lags], np.float64)
    H = sfft.rfft(h)
    m = np.arange(Nu)
    uh = (m - (g.Nu - 1) / 2.0) * g.Du
    C = fdk_scale(g)
    out = np.empty((n_views, n_rows, Nu), np.float64)
    for r0 in range(n_rows):
        v = v0 + r0
        vh = (v - (g.Nv - 1) / 2.0) * g.Dv
        Fcos = g.D / np.sqrt(g.D * g.D + uh * uh + vh * vh)
        rows = E[:, r0, :].astype(np.float64) * Fcos[None, :]
        spec = sfft.rfft(rows, n=L, axis=1, workers=workers)
        out[:, r0, :] = C * sfft.irfft(spec * H[None, :], n=L, axis=1, workers=workers)[:, :Nu]
    return out


def interp2(g: OracleGeometry, Q: np.ndarray, u: float, v: float, v0: int = 0):
    """Alg. alg:subpixel on one filtered view Q ([n_rows][Nu], rows v0..)."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    miss = ctypes.c_int(0)
    cg = g.c()
    val = _L().oracle_interp2(ctypes.byref(cg), _ptr(Q, ctypes.c_double), int(v0), Q.shape[0],
                              float(u), float(v), ctypes.byref(miss))
    return float(val), bool(miss.value)


class BandError(RuntimeError):
    pass


def backproject(g: OracleGeometry, Q: np.ndarray, ijk: np.ndarray, s0: int = 0,
                v0: int = 0) -> np.ndarray:
    """Alg. alg:bp for a voxel list ijk (n x 3 int).  Q: [n_views][n_rows][Nu] fp64."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    ijk = np.ascontiguousarray(ijk, dtype=np.int32).reshape(-1, 3)
    out = np.empty(ijk.shape[0], np.float64)
    cg = g.c()
    st = _L().oracle_backproject(ctypes.byref(cg), _ptr(Q, ctypes.c_double), int(s0), Q.shape[0],
                                 int(v0), Q.shape[1], ijk.shape[0], _ptr(ijk, ctypes.c_int),
                                 _ptr(out, ctypes.c_double))
    if st != 0:
        raise BandError("a tap inside the detector is outside the supplied row band")
    return out


def backproject_volume(g: OracleGeometry, Q: np.ndarray, s0: int = 0, v0: int = 0,
                       k0: int = 0, nk: int | None = None) -> np.ndarray:
    """Alg. alg:bp over the k-slab k0..k0+nk-1: returns [nk][Ny][Nx] fp64."""
    if nk is None:
        nk = g.Nz - k0
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    out = np.empty((nk, g.Ny, g.Nx), np.float64)
    cg = g.c()
    st = _L().oracle_backproject_volume(ctypes.byref(cg), _ptr(Q, ctypes.c_double), int(s0),
                                        Q.shape[0], int(v0), Q.shape[1], int(k0), int(nk),
                                        _ptr(out, ctypes.c_double))
    if st != 0:
        raise BandError("a tap inside the detector is outside the supplied row band")
    return out


def reconstruct(g: OracleGeometry, E: np.ndarray, s0: int = 0, fft: bool = False) -> np.ndarray:
    """FDK = Alg. alg:filter then Alg. alg:bp over the whole volume ([Nz][Ny][Nx] fp64)."""
    Q = filter_fft(g, E) if fft else filter_direct(g, E)
    return backproject_volume(g, Q, s0=s0)


def forward_project(g: OracleGeometry, vol: np.ndarray, s0: int = 0, n_views: int = 1,
                    v0: int = 0, n_rows: int | None = None, k0: int = 0) -> np.ndarray:
    """The matched forward projector (reading c-I1, the transpose of Alg. alg:bp +
    alg:subpixel) of the slab vol [nk][Ny][Nx] (k0..): returns [n_views][n_rows][Nu] fp64."""
    if n_rows is None:
        n_rows = g.Nv - v0
    vol = np.ascontiguousarray(vol, dtype=np.float64)
    out = np.empty((n_views, n_rows, g.Nu), np.float64)
    cg = g.c()
    st = _L().oracle_forward_project(ctypes.byref(cg), _ptr(vol, ctypes.c_double), int(k0),
                                     vol.shape[0], int(s0), int(n_views), int(v0), int(n_rows),
                                     _ptr(out, ctypes.c_double))
    if st != 0:
        raise BandError("a tap on the detector is outside the supplied row band")
    return out


def sart(g: OracleGeometry, b: np.ndarray, n_iter: int, lam: float = 1.0,
         block: int | None = None, x0: np.ndarray | None = None,
         nonneg: bool = False) -> np.ndarray:
    """SART / SIRT (Andersen & Kak, cited at P:266; reading c-I2), written out step by step:
    for each iteration and each subset S of `block` consecutive views (block = all views:
    SIRT),  x <- x + lam * M_S^T((b_S - M_S x) / R_S) / C_S  with R_S = M_S 1 (row sums),
    C_S = M_S^T 1 (column sums), M_S the forward projector of the views of S and M_S^T the
    back-projector (Alg. alg:bp).  Zero normalisers leave the term out (reading c-I3).
    b: [Np][Nv][Nu] for views 0..Np-1.  Returns x [Nz][Ny][Nx] fp64."""
    Np = b.shape[0]
    block = block or Np
    x = np.zeros((g.Nz, g.Ny, g.Nx)) if x0 is None else np.array(x0, dtype=np.float64)
    ones_vol = np.ones((g.Nz, g.Ny, g.Nx))
    for _ in range(n_iter):
        for s0 in range(0, Np, block):
            n = min(block, Np - s0)
            R = forward_project(g, ones_vol, s0, n)
            C = backproject_volume(g, np.ones((n, g.Nv, g.Nu)), s0=s0)
            resid = b[s0:s0 + n] - forward_project(g, x, s0, n)
            ratio = np.where(R > 0, resid / np.where(R > 0, R, 1.0), 0.0)
            c = backproject_volume(g, ratio, s0=s0)
            x = x + np.where(C > 0, lam * c / np.where(C > 0, C, 1.0), 0.0)
            if nonneg:
                x = np.maximum(x, 0.0)
    return x


def mlem(g: OracleGeometry, b: np.ndarray, n_iter: int, block: int | None = None,
         x0: np.ndarray | None = None) -> np.ndarray:
    """MLEM / OS-EM (Shepp & Vardi, cited at P:266; reading c-I4), step by step: for each
    iteration and subset S,  x <- x * M_S^T(b_S / M_S x) / C_S  with C_S = M_S^T 1; a ray the
    estimate does not reach (M_S x = 0) contributes 0, a voxel no ray sees (C_S = 0) is kept.
    x0 defaults to 1 everywhere.  b: [Np][Nv][Nu].  Returns x [Nz][Ny][Nx] fp64."""
    Np = b.shape[0]
    block = block or Np
    x = np.ones((g.Nz, g.Ny, g.Nx)) if x0 is None else np.array(x0, dtype=np.float64)
    for _ in range(n_iter):
        for s0 in range(0, Np, block):
            n = min(block, Np - s0)
            C = backproject_volume(g, np.ones((n, g.Nv, g.Nu)), s0=s0)
            ax = forward_project(g, x, s0, n)
            ratio = np.where(ax > 0, b[s0:s0 + n] / np.where(ax > 0, ax, 1.0), 0.0)
            c = backproject_volume(g, ratio, s0=s0)
            x = np.where(C > 0, x * c / np.where(C > 0, C, 1.0), x)
    return x
