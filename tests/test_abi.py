"""The C-ABI library loads, exports every symbol include/ifdk.h declares, and its
host-only geometry functions behave (no GPU needed)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "ifdk.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ifdk_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1909_02724_b200 import build, ifdk

    assert os.path.exists(build.LIB)
    lib = ctypes.CDLL(build.LIB)
    syms = _header_symbols()
    assert set(syms) == set(ifdk.EXPORTS), syms
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a():
    import subprocess

    from paper_1909_02724_b200 import build

    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_geometry_validation():
    from paper_1909_02724_b200 import Geometry, IfdkError

    ok = dict(Nu=16, Nv=16, Nx=8, Ny=8, Nz=8, Du=1.0, Dv=1.0, Dx=1.0, Dy=1.0, Dz=1.0, D=40.0,
              d=25.0, theta=0.1)
    Geometry(**ok)
    for k, v in (("Nu", 0), ("Dx", 0.0), ("Dv", -1.0), ("D", 20.0), ("d", 0.0),
                 ("theta", float("nan")), ("theta", 0.0)):
        with pytest.raises(IfdkError) as e:
            Geometry(**{**ok, k: v})
        assert e.value.status == 1, (k, v)
    with pytest.raises(IfdkError) as e:  # volume reaches the source circle
        Geometry(**{**ok, "Dx": 6.0, "Dy": 6.0})
    assert e.value.status == 2


def test_projection_matrix_matches_oracle():
    """libifdk assembles P from closed forms; the oracle multiplies the printed
    matrices.  Two independent derivations of P:15-82 must agree."""
    import oracle
    from paper_1909_02724_b200 import Geometry

    rng = np.random.default_rng(1)
    for _ in range(50):
        Nx, Ny, Nz = (int(x) for x in rng.integers(4, 400, 3))
        Nu, Nv = (int(x) for x in rng.integers(8, 800, 2))
        d = float(rng.uniform(300, 1500))
        args = dict(Nu=Nu, Nv=Nv, Nx=Nx, Ny=Ny, Nz=Nz, Du=float(rng.uniform(0.1, 1)),
                    Dv=float(rng.uniform(0.1, 1)), Dx=float(rng.uniform(0.05, 0.4)),
                    Dy=float(rng.uniform(0.05, 0.4)), Dz=float(rng.uniform(0.05, 0.4)),
                    D=d * float(rng.uniform(1.1, 2)), d=d, theta=float(rng.uniform(0.001, 0.5)))
        g = Geometry(**args)
        og = oracle.OracleGeometry(**args)
        for s in rng.integers(-10, 5000, 4):
            P1, P2 = g.projection_matrix(int(s)), oracle.projection_matrix(og, int(s))
            scale = np.abs(P2).max(axis=1, keepdims=True)
            assert np.all(np.abs(P1 - P2) <= 1e-13 * scale)
            assert P1[0, 2] == 0.0 and P1[2, 2] == 0.0


def test_band_rows_cover_every_tap():
    """ifdk_band_rows must contain every detector row any voxel of the slab taps
    (rows floor(v) and floor(v)+1, oracle P), for every view."""
    import oracle
    import synth
    from paper_1909_02724_b200 import Geometry

    spec = synth.ConfigSpec("band", 90, 64, 48, 40, 36, 50)
    g = Geometry.from_spec(spec)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ii, jj = np.meshgrid(np.arange(spec.Nx), np.arange(spec.Ny), indexing="ij")
    for k0, nk in ((0, 50), (0, 13), (13, 20), (49, 1)):
        for s in range(0, 90, 7):
            lo, hi = g.band_rows(k0, nk, s)
            P = oracle.projection_matrix(og, s)
            for k in (k0, k0 + nk - 1):
                x = P[1, 0] * ii + P[1, 1] * jj + P[1, 2] * k + P[1, 3]
                z = P[2, 0] * ii + P[2, 1] * jj + P[2, 3]
                nv = np.floor(x / z)
                need_lo = max(int(nv.min()), 0)
                need_hi = min(int(nv.max()) + 1, spec.Nv - 1)
                assert lo <= need_lo and hi >= need_hi, (k0, nk, s, lo, hi, need_lo, need_hi)


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    from paper_1909_02724_b200 import Geometry, IfdkError, ifdk_reconstruct_host

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = Geometry(16, 16, 8, 8, 8, 1.0, 1.0, 1.0, 1.0, 1.0, 40.0, 25.0, 0.1)
    raw = np.zeros((2, 16, 16), np.float32)
    vol = np.zeros((8, 8, 8), np.float32)
    with pytest.raises(IfdkError) as e:
        ifdk_reconstruct_host(g, raw, vol, stream=0)
    assert e.value.status == 4


def test_iterative_entry_points_validate_and_fail_loudly_without_gpu():
    """ifdk_forward_project / ifdk_sart_* / ifdk_fill: argument errors before any device work,
    then IFDK_ERR_CUDA without a GPU (no CPU fallback)."""
    import ctypes

    import torch

    from paper_1909_02724_b200 import Geometry, ifdk

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = ifdk._lib
    g = Geometry(16, 16, 8, 8, 8, 1.0, 1.0, 1.0, 1.0, 1.0, 40.0, 25.0, 0.1)
    fake = ctypes.c_void_p(0x1000)
    # band too small for the slab -> SHAPE; accumulate 2 -> INVALID_ARGUMENT
    assert lib.ifdk_forward_project(g.handle, fake, 0, 8, 0, 2, fake, 7, 1, 0, None) == 3
    assert lib.ifdk_forward_project(g.handle, fake, 0, 8, 0, 2, fake, 0, 16, 2, None) == 1
    assert lib.ifdk_forward_project(g.handle, fake, 0, 9, 0, 2, fake, 0, 16, 0, None) == 3
    assert lib.ifdk_forward_project(g.handle, fake, 0, 8, 0, 2, fake, 0, 16, 0, None) == 4
    assert lib.ifdk_sart_update(fake, fake, fake, ctypes.c_float(2.0), 10, 0, None) == 1
    assert lib.ifdk_sart_update(fake, fake, fake, ctypes.c_float(1.0), -1, 0, None) == 3
    assert lib.ifdk_sart_update(fake, fake, fake, ctypes.c_float(1.0), 10, 0, None) == 4
    assert lib.ifdk_sart_ratio(fake, None, fake, fake, 10, None) == 1
    assert lib.ifdk_sart_ratio(fake, fake, fake, fake, 10, None) == 4
    assert lib.ifdk_fill(fake, ctypes.c_float(1.0), 10, None) == 4
