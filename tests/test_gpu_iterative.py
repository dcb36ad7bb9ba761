"""GPU parity of the iterative-reconstruction path through the C ABI:
the matched forward projector against the fp64 oracle element by element, its adjoint
relation to BP-sm100, the element-wise SART steps against their definitions, and SART /
SIRT iterations against the oracle's, on seeded inputs."""
import numpy as np
import pytest

import oracle
import synth
from parity_util import VOL_MAX_REL, VOL_RMSE, assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _spec(Np, Nu, Nv, Nx, Ny, Nz, **kw):
    return synth.ConfigSpec(f"{Np}x{Nu}x{Nv}->{Nx}x{Ny}x{Nz}", Np, Nu, Nv, Nx, Ny, Nz, **kw)


def _volume(spec, seed=0):
    """A seeded fp32 test volume: the voxelised phantom (ellipsoid indicator sums at voxel
    centres) plus uniform noise, so every voxel is non-zero."""
    rng = np.random.default_rng(seed)
    return (synth.phantom_volume(spec) + rng.uniform(0.0, 0.1, (spec.Nz, spec.Ny, spec.Nx))
            ).astype(np.float32)


def _fp_case(torch, spec, s0, n, k0, nk, v0=None, n_rows=None, base=None, seed=0):
    from paper_1909_02724_b200 import Geometry, ifdk_forward_project

    g = Geometry.from_spec(spec)
    if v0 is None:
        v0, n_rows = 0, spec.Nv
    vol = _volume(spec, seed)[k0:k0 + nk].copy()
    proj = torch.zeros((n, n_rows, spec.Nu), device="cuda")
    if base is not None:
        proj.copy_(torch.from_numpy(base))
    ifdk_forward_project(g, torch.from_numpy(vol).cuda(), s0, proj, k0=k0, v0=v0,
                         accumulate=base is not None)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.forward_project(og, vol.astype(np.float64), s0, n, v0=v0, n_rows=n_rows, k0=k0)
    if base is not None:
        ref = ref + base
    return proj.cpu().numpy(), ref


def test_fp_config1(torch_cuda):
    spec = synth.config(1)
    got, ref = _fp_case(torch_cuda, spec, 0, 64, 0, 64)
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, "fp config 1")


def test_fp_ragged_slab_band_and_accumulate(torch_cuda):
    """Nx, Ny not multiples of the 16x16 tile, an unaligned slab, a view offset, a detector row
    band covering the slab's footprint, and accumulation onto existing projections."""
    from paper_1909_02724_b200 import Geometry

    spec = _spec(150, 80, 72, 37, 23, 150)
    g = Geometry.from_spec(spec)
    s0, n, k0, nk = 17, 29, 45, 90
    lo = min(g.band_rows(k0, nk, s)[0] for s in range(s0, s0 + n))
    hi = max(g.band_rows(k0, nk, s)[1] for s in range(s0, s0 + n))
    # a base of the projections' own magnitude (~1e-5: W = 1/z^2), so that fp32 addition onto
    # it keeps the forward projection's digits
    _, ref0 = _fp_case(torch_cuda, spec, s0, n, k0, nk, v0=lo, n_rows=hi - lo + 1)
    base = (np.random.default_rng(3).standard_normal((n, hi - lo + 1, spec.Nu))
            * np.abs(ref0).max()).astype(np.float32)
    got, ref = _fp_case(torch_cuda, spec, s0, n, k0, nk, v0=lo, n_rows=hi - lo + 1, base=base)
    assert_parity(got - base, ref - base, VOL_RMSE, VOL_MAX_REL, "fp ragged")


def test_fp_truncated_detector(torch_cuda):
    """A detector smaller than the volume's shadow: taps off the detector are dropped (c-A9)."""
    spec = _spec(40, 24, 20, 32, 32, 40, det_mm=120.0)
    got, ref = _fp_case(torch_cuda, spec, 0, 40, 0, 40)
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, "fp truncated")


def test_fp_is_adjoint_of_bp_on_gpu(torch_cuda):
    """<M x, y> = <x, M^T y> with both operators on the GPU (fp32; dot products in fp64)."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, ifdk_forward_project

    spec = _spec(96, 128, 128, 96, 80, 96)
    g = Geometry.from_spec(spec)
    rng = np.random.default_rng(21)
    x = rng.standard_normal((spec.Nz, spec.Ny, spec.Nx)).astype(np.float32)
    y = rng.standard_normal((spec.Np, spec.Nv, spec.Nu)).astype(np.float32)
    Mx = torch.empty((spec.Np, spec.Nv, spec.Nu), device="cuda")
    ifdk_forward_project(g, torch.from_numpy(x).cuda(), 0, Mx)
    MTy = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_backproject(g, torch.from_numpy(y).cuda(), 0, MTy)
    lhs = float((Mx.cpu().numpy().astype(np.float64) * y).sum())
    rhs = float((x.astype(np.float64) * MTy.cpu().numpy()).sum())
    scale = float(np.abs(Mx.cpu().numpy().astype(np.float64) * y).sum())
    print(f"ADJOINT <Mx,y>={lhs:.9e} <x,MTy>={rhs:.9e} |diff|/sum|terms|={abs(lhs - rhs) / scale:.2e}")
    assert abs(lhs - rhs) <= 1e-6 * scale


def test_sart_elementwise_steps_match_definitions(torch_cuda):
    torch = torch_cuda
    from paper_1909_02724_b200 import ifdk_fill, ifdk_sart_ratio, ifdk_sart_update

    rng = np.random.default_rng(2)
    n = 100003
    b, ax, c = (rng.standard_normal(n).astype(np.float32) for _ in range(3))
    R = rng.uniform(-0.2, 2.0, n).astype(np.float32)
    C = rng.uniform(-0.2, 2.0, n).astype(np.float32)
    x = rng.standard_normal(n).astype(np.float32)
    dev = {k: torch.from_numpy(v).cuda() for k, v in dict(b=b, ax=ax, R=R, C=C, c=c, x=x).items()}
    out = torch.empty(n, device="cuda")
    ifdk_sart_ratio(dev["b"], dev["ax"], dev["R"], out)
    ref = np.where(R > 0, (b - ax) / np.where(R > 0, R, np.float32(1)), np.float32(0))
    assert np.array_equal(out.cpu().numpy(), ref)
    ifdk_sart_update(dev["x"], dev["c"], dev["C"], 0.75, nonneg=True)
    lam = np.float32(0.75)
    ref = np.maximum(x + np.where(C > 0, lam * c / np.where(C > 0, C, np.float32(1)),
                                  np.float32(0)), np.float32(0))
    assert np.array_equal(dev["x"].cpu().numpy(), ref)
    ifdk_fill(out, 1.5)
    assert bool((out == 1.5).all())


@pytest.mark.parametrize("block,n_iter,lam", [(8, 2, 1.0), (None, 3, 1.5)])
def test_sart_matches_oracle(torch_cuda, block, n_iter, lam):
    """OS-SART (8-view subsets) and SIRT (all views) on the GPU vs the oracle's SART, same
    measured projections (the oracle's forward projection of the seeded volume, fp32)."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, sart

    spec = _spec(32, 48, 48, 40, 40, 40)
    og = oracle.OracleGeometry(**spec.geometry_args())
    b = oracle.forward_project(og, _volume(spec, 5).astype(np.float64), 0, spec.Np)
    b32 = b.astype(np.float32)
    x = sart(Geometry.from_spec(spec), torch.from_numpy(b32).cuda(), n_iter, lam=lam, block=block)
    ref = oracle.sart(og, b32.astype(np.float64), n_iter, lam=lam, block=block)
    assert_parity(x.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, f"sart block={block}")


def test_fp_config3_full_size_slab(torch_cuda):
    """Config 3's full detector and volume extent (1024^2 detector, 1024 x 1024 columns) in
    the slab launch configuration: a 64-slice slab through the phantom's centre projected into
    the row band it reaches, for 3 views spread over the circle; every band pixel compared."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_forward_project

    spec = synth.config(3)
    g = Geometry.from_spec(spec)
    og = oracle.OracleGeometry(**spec.geometry_args())
    k0, nk = 480, 64
    vol = synth.phantom_volume(spec, k0, nk).astype(np.float32)
    dvol = torch.from_numpy(vol).cuda()
    for s in (0, 301, 777):
        lo, hi = g.band_rows(k0, nk, s)
        proj = torch.empty((1, hi - lo + 1, spec.Nu), device="cuda")
        ifdk_forward_project(g, dvol, s, proj, k0=k0, v0=lo)
        ref = oracle.forward_project(og, vol.astype(np.float64), s, 1, v0=lo,
                                     n_rows=hi - lo + 1, k0=k0)
        assert_parity(proj.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, f"fp config 3 slab view {s}")


def test_mlem_elementwise_steps_match_definitions(torch_cuda):
    torch = torch_cuda
    from paper_1909_02724_b200 import ifdk_mlem_ratio, ifdk_mlem_update

    rng = np.random.default_rng(4)
    n = 70001
    b = rng.uniform(0, 2, n).astype(np.float32)
    ax = rng.uniform(-0.1, 2, n).astype(np.float32)
    x = rng.uniform(0.1, 1, n).astype(np.float32)
    c = rng.uniform(0, 2, n).astype(np.float32)
    C = rng.uniform(-0.1, 2, n).astype(np.float32)
    out = torch.empty(n, device="cuda")
    ifdk_mlem_ratio(torch.from_numpy(b).cuda(), torch.from_numpy(ax).cuda(), out)
    ref = np.where(ax > 0, b / np.where(ax > 0, ax, np.float32(1)), np.float32(0))
    assert np.array_equal(out.cpu().numpy(), ref)
    xd = torch.from_numpy(x).cuda()
    ifdk_mlem_update(xd, torch.from_numpy(c).cuda(), torch.from_numpy(C).cuda())
    ref = np.where(C > 0, x * c / np.where(C > 0, C, np.float32(1)), x)
    assert np.array_equal(xd.cpu().numpy(), ref)


@pytest.mark.parametrize("block,n_iter", [(8, 2), (None, 3)])
def test_mlem_matches_oracle(torch_cuda, block, n_iter):
    """OS-EM (8-view subsets) and MLEM on the GPU vs the oracle's, same measured projections."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, mlem

    spec = _spec(32, 48, 48, 40, 40, 40)
    og = oracle.OracleGeometry(**spec.geometry_args())
    b32 = oracle.forward_project(og, _volume(spec, 6).astype(np.float64), 0, spec.Np).astype(np.float32)
    x = mlem(Geometry.from_spec(spec), torch.from_numpy(b32).cuda(), n_iter, block=block)
    ref = oracle.mlem(og, b32.astype(np.float64), n_iter, block=block)
    assert_parity(x.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, f"mlem block={block}")


def test_fp_many_detector_rows_per_slice(torch_cuda):
    """The projector's large-dv walk (1.9-3.3 detector rows per slice; larger patches exceed its
    shared memory and are refused): per-column fp64 invariants with dv split into whole rows +
    an fp32 fraction, as the back-projector's single-slice walk."""
    spec = _spec(35, 21, 49, 14, 33, 62, d=1035.113914283941, D=1384.110376984815,
                 det_mm=180.43609777816965, cube_mm=409.8307371445136)
    got, ref = _fp_case(torch_cuda, spec, 0, 35, 0, 62)
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, "fp 1.9-3.3 detector rows per slice")
