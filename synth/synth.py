"""Workload recipe + analytic phantom projections (see synth/__init__.py)."""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_CU_SRC = os.path.join(_HERE, "synth_cuda.cu")
_CU_LIB = os.path.join(_HERE, "libsynth_cuda.so")


def build(force: bool = False, cuda: bool = True) -> None:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99", _SRC,
                               "-o", _LIB, "-lm"])
    if cuda and (force or not os.path.exists(_CU_LIB)
                 or os.path.getmtime(_CU_LIB) < os.path.getmtime(_CU_SRC)):
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-Xcompiler", "-fPIC", "-shared", _CU_SRC, "-o", _CU_LIB])


# --------------------------------------------------------------------------- recipe
@dataclass(frozen=True)
class ConfigSpec:
    """One BASELINE.json config: Np views of Nu x Nv -> Nx x Ny x Nz, plus the
    scanner geometry fixed in DESIGN.md (the paper gives none, reading c-A16):
    D = 1536 mm, d = 1024 mm, a 400 mm square detector, a 180 mm cube."""

    name: str
    Np: int
    Nu: int
    Nv: int
    Nx: int
    Ny: int
    Nz: int
    D: float = 1536.0
    d: float = 1024.0
    det_mm: float = 400.0
    cube_mm: float = 180.0

    @property
    def Du(self) -> float:
        return self.det_mm / self.Nu

    @property
    def Dv(self) -> float:
        return self.det_mm / self.Nv

    @property
    def Dx(self) -> float:
        return self.cube_mm / self.Nx

    @property
    def Dy(self) -> float:
        return self.cube_mm / self.Ny

    @property
    def Dz(self) -> float:
        return self.cube_mm / self.Nz

    @property
    def theta(self) -> float:
        return 2.0 * math.pi / self.Np  # theta = 2 pi / Np

    @property
    def updates(self) -> int:
        return self.Nx * self.Ny * self.Nz * self.Np

    def geometry_args(self) -> dict:
        return dict(Nu=self.Nu, Nv=self.Nv, Nx=self.Nx, Ny=self.Ny, Nz=self.Nz, Du=self.Du,
                    Dv=self.Dv, Dx=self.Dx, Dy=self.Dy, Dz=self.Dz, D=self.D, d=self.d,
                    theta=self.theta)


CONFIGS = {
    1: ConfigSpec("64x64^2->64^3", 64, 64, 64, 64, 64, 64),
    2: ConfigSpec("512x512^2->512^3", 512, 512, 512, 512, 512, 512),
    3: ConfigSpec("1024x1024^2->1024^3", 1024, 1024, 1024, 1024, 1024, 1024),
    4: ConfigSpec("2048x2048^2->2048^3", 2048, 2048, 2048, 2048, 2048, 2048),
    5: ConfigSpec("4096x2048^2->4096^3", 4096, 2048, 2048, 4096, 4096, 4096),
}


def config(n: int) -> ConfigSpec:
    return CONFIGS[n]


# Ten ellipsoids, normalised units: (a, b, c, x0, y0, z0, phi_deg, rho).  A
# modified-contrast 3-D Shepp-Logan variant with z-rotation only; the paper only
# names the phantom, so this table is the builder's choice.
PHANTOM_TABLE = (
    (0.69, 0.92, 0.90, 0.0, 0.0, 0.0, 0.0, 1.0),
    (0.6624, 0.874, 0.88, 0.0, -0.0184, 0.0, 0.0, -0.8),
    (0.11, 0.31, 0.22, 0.22, 0.0, 0.0, -18.0, -0.2),
    (0.16, 0.41, 0.28, -0.22, 0.0, 0.0, 18.0, -0.2),
    (0.21, 0.25, 0.41, 0.0, 0.35, -0.15, 0.0, 0.1),
    (0.046, 0.046, 0.05, 0.0, 0.1, 0.25, 0.0, 0.1),
    (0.046, 0.046, 0.05, 0.0, -0.1, 0.25, 0.0, 0.1),
    (0.046, 0.023, 0.05, -0.08, -0.605, 0.0, 0.0, 0.1),
    (0.023, 0.023, 0.02, 0.0, -0.606, 0.0, 0.0, 0.1),
    (0.023, 0.046, 0.02, 0.06, -0.605, 0.0, 0.0, 0.1),
)


def ellipsoids(half_extent_mm: float, table=PHANTOM_TABLE) -> np.ndarray:
    """Ellipsoid records (n x 10 fp64) scaled to a unit half-extent of
    ``half_extent_mm`` (0.9 x the cube half-side for the configs)."""
    rec = []
    for a, b, c, x0, y0, z0, phi, rho in table:
        p = math.radians(phi)
        s = half_extent_mm
        rec.append([x0 * s, y0 * s, z0 * s, a * s, b * s, c * s, math.cos(p), math.sin(p), rho, 0.0])
    return np.asarray(rec, np.float64)


def default_ellipsoids(spec: ConfigSpec) -> np.ndarray:
    return ellipsoids(0.9 * spec.cube_mm / 2.0)


class _Scanner(ctypes.Structure):
    _fields_ = [("Nu", ctypes.c_int), ("Nv", ctypes.c_int), ("Du", ctypes.c_double),
                ("Dv", ctypes.c_double), ("D", ctypes.c_double), ("d", ctypes.c_double),
                ("theta", ctypes.c_double)]


def _scanner(Nu, Nv, Du, Dv, D, d, theta) -> _Scanner:
    return _Scanner(int(Nu), int(Nv), float(Du), float(Dv), float(D), float(d), float(theta))


_lib = None
_culib = None


def _L():
    global _lib
    if _lib is None:
        build(cuda=False)
        _lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        _lib.synth_project.argtypes = [ctypes.POINTER(_Scanner), dp, ctypes.c_int, ctypes.c_long,
                                       ctypes.c_long, ctypes.c_int, ctypes.c_int, fp]
        _lib.synth_density.argtypes = [dp, ctypes.c_int, ctypes.c_long, dp, dp]
        _lib.synth_add_noise.argtypes = [fp, ctypes.c_long, ctypes.c_long, ctypes.c_uint64,
                                         ctypes.c_double]
    return _lib


def project(Nu, Nv, Du, Dv, D, d, theta, ell: np.ndarray, s0: int, n_views: int, v0: int = 0,
            n_rows: int | None = None) -> np.ndarray:
    """Analytic line integrals through pixel centres: E [n_views][n_rows][Nu] fp32."""
    if n_rows is None:
        n_rows = Nv - v0
    ell = np.ascontiguousarray(ell, np.float64)
    E = np.empty((n_views, n_rows, Nu), np.float32)
    sc = _scanner(Nu, Nv, Du, Dv, D, d, theta)
    _L().synth_project(ctypes.byref(sc), ell.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                       ell.shape[0], int(s0), int(n_views), int(v0), int(n_rows),
                       E.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    return E


def project_gpu(Nu, Nv, Du, Dv, D, d, theta, ell: np.ndarray, s0: int, n_views: int, v0: int,
                n_rows: int, out_ptr: int, stream: int = 0) -> None:
    """Same as ``project`` but on the GPU into a device buffer (fp64 arithmetic).
    Used by bench.py to make config-4/5 inputs; pinned to ``project`` by a GPU test."""
    global _culib
    if _culib is None:
        if not os.path.exists(_CU_LIB):
            raise RuntimeError(f"{_CU_LIB} missing: run __graft_entry__.build()")
        _culib = ctypes.CDLL(_CU_LIB)
        _culib.synth_project_cuda.argtypes = [ctypes.POINTER(_Scanner), ctypes.c_void_p,
                                              ctypes.c_int, ctypes.c_long, ctypes.c_long,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                              ctypes.c_void_p]
        _culib.synth_project_cuda.restype = ctypes.c_int
    ell = np.ascontiguousarray(ell, np.float64)
    sc = _scanner(Nu, Nv, Du, Dv, D, d, theta)
    rc = _culib.synth_project_cuda(ctypes.byref(sc), ell.ctypes.data, ell.shape[0], int(s0),
                                   int(n_views), int(v0), int(n_rows), ctypes.c_void_p(out_ptr),
                                   ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"synth_project_cuda failed: {rc}")


def voxel_world(spec_or_g, i, j, k):
    """World coordinates (mm) of voxel centres (reading c-A15)."""
    g = spec_or_g
    cx, cy, cz = (g.Nx - 1) / 2.0, (g.Ny - 1) / 2.0, (g.Nz - 1) / 2.0
    return (g.Dx * (np.asarray(i) - cx), -g.Dy * (np.asarray(j) - cy), -g.Dz * (np.asarray(k) - cz))


def density(ell: np.ndarray, xyz: np.ndarray) -> np.ndarray:
    xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
    ell = np.ascontiguousarray(ell, np.float64)
    out = np.empty(xyz.shape[0], np.float64)
    dp = ctypes.POINTER(ctypes.c_double)
    _L().synth_density(ell.ctypes.data_as(dp), ell.shape[0], xyz.shape[0], xyz.ctypes.data_as(dp),
                       out.ctypes.data_as(dp))
    return out


def phantom_volume(spec: ConfigSpec, k0: int = 0, nk: int | None = None) -> np.ndarray:
    """The phantom's density sampled at the voxel centres of slices k0..k0+nk-1,
    [nk][Ny][Nx] fp64: a structured test volume for the forward projector (no method
    arithmetic)."""
    nk = spec.Nz - k0 if nk is None else nk
    k, j, i = np.meshgrid(np.arange(k0, k0 + nk), np.arange(spec.Ny), np.arange(spec.Nx),
                          indexing="ij")
    X, Y, Z = voxel_world(spec, i.ravel(), j.ravel(), k.ravel())
    rho = density(default_ellipsoids(spec), np.stack([X, Y, Z], axis=1))
    return rho.reshape(nk, spec.Ny, spec.Nx)


def add_noise(E: np.ndarray, sigma: float, seed: int = 1234, base: int = 0) -> np.ndarray:
    """E + sigma * N(0,1) from a counter-based generator (in place on a copy)."""
    out = np.ascontiguousarray(E, np.float32).copy()
    _L().synth_add_noise(out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), out.size, int(base),
                         int(seed) & 0xFFFFFFFFFFFFFFFF, float(sigma))
    return out
