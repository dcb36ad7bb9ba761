"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle, element by element,
on the same seeded inputs (sizes the oracle finishes in seconds; several tiles and
ragged tails), plus edge cases and bitwise invariants."""
import math

import numpy as np
import pytest

import oracle
import synth
from parity_util import Q_MAX_REL, Q_RMSE, VOL_MAX_REL, VOL_RMSE, assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture
def auto_variant():
    """Restores the automatic BP walk after a test that pins one (ifdk_set_bp_variant)."""
    yield
    from paper_1909_02724_b200 import set_bp_variant

    set_bp_variant(0, 0)


def _spec(Np, Nu, Nv, Nx, Ny, Nz, **kw):
    return synth.ConfigSpec(f"{Np}x{Nu}x{Nv}->{Nx}x{Ny}x{Nz}", Np, Nu, Nv, Nx, Ny, Nz, **kw)


def _phantom_E(spec, s0=0, n=None, v0=0, n_rows=None):
    n = spec.Np if n is None else n
    ell = synth.default_ellipsoids(spec)
    return synth.project(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, s0,
                         n, v0, n_rows)


def _oracle_Q32(spec, E, v0=0):
    """Filtered views computed by the oracle, rounded to fp32: a seeded BP input that never
    touches the CUDA path."""
    og = oracle.OracleGeometry(**spec.geometry_args())
    return oracle.filter_fft(og, E, v0=v0).astype(np.float32)


# ------------------------------------------------------------------------------- filter
@pytest.mark.parametrize("Nu,n_rows,n_views,v0", [
    (64, 64, 5, 0),      # odd number of rows overall: the last complex pair is half empty
    (100, 30, 3, 7),     # Nu not a power of two: L = 256
    (37, 5, 1, 0),       # odd Nu, a single view
    (512, 8, 4, 200),    # a row band in the middle of the detector
    (2048, 3, 2, 1000),  # L = 4096, the config-4/5 row length
    (2100, 2, 3, 0),     # Nu > 2048: the generic Stockham kernel (L = 8192)
])
def test_filter_matches_oracle(torch_cuda, Nu, n_rows, n_views, v0):
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_filter

    Nv = max(v0 + n_rows + 3, 16)
    spec = _spec(90, Nu, Nv, 32, 32, 32)
    g = Geometry.from_spec(spec)
    rng = np.random.default_rng(Nu + n_rows)
    E = (np.abs(rng.standard_normal((n_views, n_rows, Nu))) * 20).astype(np.float32)
    raw = torch.from_numpy(E).cuda()
    out = torch.empty_like(raw)
    ifdk_filter(g, raw, out, v0=v0)
    Qref = oracle.filter_direct(oracle.OracleGeometry(**spec.geometry_args()), E, v0=v0)
    assert_parity(out.cpu().numpy(), Qref, Q_RMSE, Q_MAX_REL, "filter")
    # in place
    ifdk_filter(g, raw, raw, v0=v0)
    assert torch.equal(raw, out)


@pytest.mark.parametrize("Nu,Nv,n_views,bands", [
    (2048, 40, 3, [(0, 39), (5, 17), (17, 30), (39, 39)]),  # f4k kernel; overlapping bands
    (100, 24, 5, [(3, 9), (0, 23)]),                          # generic kernel, odd row total
])
def test_filter_scatter_equals_filter_then_slice(torch_cuda, Nu, Nv, n_views, bands):
    """The fused filter + band scatter (the k-slab exchange riding the filter) stores exactly
    ifdk_filter's values, row band by row band, and nothing else."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_filter, ifdk_filter_scatter

    spec = _spec(64, Nu, Nv, 32, 32, 32)
    g = Geometry.from_spec(spec)
    rng = np.random.default_rng(Nu)
    raw = torch.from_numpy((np.abs(rng.standard_normal((n_views, Nv, Nu))) * 20)
                           .astype(np.float32)).cuda()
    Q = torch.empty_like(raw)
    ifdk_filter(g, raw, Q)
    outs = [torch.full((n_views, hi - lo + 1, Nu), float("nan"), device="cuda")
            for lo, hi in bands]
    ifdk_filter_scatter(g, raw, [(o.data_ptr(), lo, hi) for o, (lo, hi) in zip(outs, bands)])
    for o, (lo, hi) in zip(outs, bands):
        assert torch.equal(o, Q[:, lo:hi + 1]), (lo, hi)


def test_filter_phantom_config1(torch_cuda):
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_filter

    spec = synth.config(1)
    E = _phantom_E(spec)
    raw = torch.from_numpy(E).cuda()
    out = torch.empty_like(raw)
    ifdk_filter(Geometry.from_spec(spec), raw, out)
    Qref = oracle.filter_direct(oracle.OracleGeometry(**spec.geometry_args()), E)
    assert_parity(out.cpu().numpy(), Qref, Q_RMSE, Q_MAX_REL, "filter config 1")


# ------------------------------------------------------------------------------- back-projection
def _bp_case(torch, spec, s0, n, k0, nk, v0=None, n_rows=None, accumulate_base=None, E=None):
    from paper_1909_02724_b200 import Geometry, ifdk_backproject

    g = Geometry.from_spec(spec)
    if v0 is None:
        v0, n_rows = 0, spec.Nv
    if E is None:
        E = _phantom_E(spec, s0, n, v0, n_rows)
    Q = _oracle_Q32(spec, E, v0)
    vol = torch.zeros((nk, spec.Ny, spec.Nx), device="cuda", dtype=torch.float32)
    if accumulate_base is not None:
        vol.copy_(torch.from_numpy(accumulate_base))
    ifdk_backproject(g, torch.from_numpy(Q).cuda(), s0, vol, k0=k0, v0=v0,
                     accumulate=accumulate_base is not None)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.backproject_volume(og, Q.astype(np.float64), s0=s0, v0=v0, k0=k0, nk=nk)
    if accumulate_base is not None:
        ref = ref + accumulate_base
    return vol.cpu().numpy(), ref


def test_bp_config1_full_volume(torch_cuda):
    got, ref = _bp_case(torch_cuda, synth.config(1), 0, 64, 0, 64)
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, "bp config 1")


def test_bp_ragged_tiles_slab_band_and_accumulate(torch_cuda):
    """Nx, Ny not multiples of the 16x16 tile, Nz not a multiple of the 64-slice chunk, an
    unaligned slab, a view offset and a detector row band; accumulate into a non-zero slab."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry

    spec = _spec(150, 80, 72, 37, 23, 150)
    g = Geometry.from_spec(spec)
    s0, n, k0, nk = 17, 29, 45, 90
    lo = min(g.band_rows(k0, nk, s)[0] for s in range(s0, s0 + n))
    hi = max(g.band_rows(k0, nk, s)[1] for s in range(s0, s0 + n))
    base = np.random.default_rng(3).standard_normal((nk, spec.Ny, spec.Nx)).astype(np.float32)
    got, ref = _bp_case(torch, spec, s0, n, k0, nk, v0=lo, n_rows=hi - lo + 1, accumulate_base=base)
    assert_parity(got - base, ref - base, VOL_RMSE, VOL_MAX_REL, "bp ragged")


def test_bp_truncated_detector_zero_border(torch_cuda):
    """A detector smaller than the volume's shadow: taps off the detector read 0 (c-A9)."""
    spec = _spec(40, 24, 20, 32, 32, 40, det_mm=120.0)
    got, ref = _bp_case(torch_cuda, spec, 0, 40, 0, 40)
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, "bp truncated")


def test_bp_global_path_nu_not_multiple_of_4(torch_cuda):
    """Nu % 4 != 0 cannot be described to TMA; the kernel reads taps from global memory."""
    spec = _spec(45, 30, 34, 20, 20, 20)
    got, ref = _bp_case(torch_cuda, spec, 3, 45, 0, 20)
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, "bp global path")


def test_bp_slab_split_is_bitwise_and_deterministic(torch_cuda):
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject

    spec = _spec(48, 96, 96, 48, 40, 200)
    g = Geometry.from_spec(spec)
    Q = torch.from_numpy(_oracle_Q32(spec, _phantom_E(spec))).cuda()
    full = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_backproject(g, Q, 0, full)
    again = torch.empty_like(full)
    ifdk_backproject(g, Q, 0, again)
    assert torch.equal(full, again)
    for cuts in ((0, 64, 200), (0, 77, 131, 200), (0, 1, 199, 200)):
        for a, b in zip(cuts[:-1], cuts[1:]):
            slab = torch.empty((b - a, spec.Ny, spec.Nx), device="cuda")
            lo = min(g.band_rows(a, b - a, s)[0] for s in range(spec.Np))
            hi = max(g.band_rows(a, b - a, s)[1] for s in range(spec.Np))
            ifdk_backproject(g, Q[:, lo:hi + 1].contiguous(), 0, slab, k0=a, v0=lo)
            assert torch.equal(slab, full[a:b]), (cuts, a, b)


def test_bp_walk_variants(torch_cuda, auto_variant):
    """PAIR walks: the fp32x2 walk on the pair patch (WALK 4), the scalar walk (2) and the RAW
    walk reading the TMA box (5) are bitwise equal, on whole chunks and on partial ones (slab
    cut inside a chunk).  TRIPLE walks: the RAW triple walk (6, the default where
    0.5 <= dv/dk) and the scalar triple walk on the pair patch (3, which serves walk 6's
    partial chunks) are bitwise equal, a slab split under walk 6 is bitwise the whole-volume
    result, and both match the oracle."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, set_bp_variant

    spec = _spec(48, 96, 160, 48, 40, 160)  # dv/dk in [0.60, 0.77]: PAIR and TRIPLE apply
    g = Geometry.from_spec(spec)
    Qn = _oracle_Q32(spec, _phantom_E(spec))
    Q = torch.from_numpy(Qn).cuda()

    def run(w, k0=0, nk=spec.Nz):
        set_bp_variant(int(w))
        vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
        ifdk_backproject(g, Q, 0, vol, k0=k0)
        torch.cuda.synchronize()
        return vol

    for walk in ("2", "5"):
        assert torch.equal(run("4"), run(walk)), walk
        assert torch.equal(run("4", 77, 54), run(walk, 77, 54)), walk
    tri = run("6")
    for w in ("3", "9", "11"):  # pair patch; TMEM accumulators: one / two views per step
        assert torch.equal(tri, run(w)), w
        assert torch.equal(run("6", 77, 54), run(w, 77, 54)), w
    for a, b in ((0, 77), (77, 131), (131, 160)):  # partial chunks at every cut
        assert torch.equal(run("6", a, b - a), tri[a:b]), (a, b)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.backproject_volume(og, Qn.astype(np.float64), s0=0, v0=0, k0=0, nk=spec.Nz)
    assert_parity(tri.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, "bp triple walk")
    assert_parity(run("4").cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, "bp pair walk")


def test_bp_three_row_triple_walk(torch_cuda, auto_variant):
    """dv/dk < 1/2 (config 5's regime): the 3-row TRIPLE RAW walk (7, the default there) and its
    pair-patch companion (8, partial chunks) are bitwise equal, slab splits are bitwise the
    whole-volume result, and the result matches the oracle."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, set_bp_variant

    spec = _spec(48, 96, 96, 48, 40, 200)  # dv/dk in [0.29, 0.37]
    g = Geometry.from_spec(spec)
    Qn = _oracle_Q32(spec, _phantom_E(spec))
    Q = torch.from_numpy(Qn).cuda()

    def run(w, k0=0, nk=spec.Nz):
        set_bp_variant(int(w))
        vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
        ifdk_backproject(g, Q, 0, vol, k0=k0)
        torch.cuda.synchronize()
        return vol

    tri = run("7")
    for w in ("8", "10", "12"):
        assert torch.equal(tri, run(w)), w
        assert torch.equal(run("7", 77, 54), run(w, 77, 54)), w
    for a, b in ((0, 77), (77, 131), (131, 200)):
        assert torch.equal(run("7", a, b - a), tri[a:b]), (a, b)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.backproject_volume(og, Qn.astype(np.float64), s0=0, v0=0, k0=0, nk=spec.Nz)
    assert_parity(tri.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, "bp 3-row triple walk")


def test_bp_view_split_accumulate_matches(torch_cuda):
    """Views in two calls (accumulate) vs one call: equal up to fp32 summation order."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject

    spec = _spec(64, 64, 64, 40, 40, 40)
    g = Geometry.from_spec(spec)
    Q = torch.from_numpy(_oracle_Q32(spec, _phantom_E(spec))).cuda()
    one = torch.empty((40, 40, 40), device="cuda")
    ifdk_backproject(g, Q, 0, one)
    two = torch.empty_like(one)
    ifdk_backproject(g, Q[:30].contiguous(), 0, two)
    ifdk_backproject(g, Q[30:].contiguous(), 30, two, accumulate=True)
    assert_parity(two.cpu().numpy(), one.cpu().numpy(), 1e-6, 1e-5, "view split")


def test_bp_long_unaligned_view_range(torch_cuda):
    """600 views from s0 = 100: the library launches per 256-view block of the global index
    (P_s in the kernel's constant parameter space).  One call equals the oracle and is
    bitwise equal to calls cut at other multiples of the 128-view summation batch."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject

    spec = _spec(900, 40, 40, 24, 20, 28)
    g = Geometry.from_spec(spec)
    s0, n = 100, 600
    Qn = _oracle_Q32(spec, _phantom_E(spec, s0, n))
    Q = torch.from_numpy(Qn).cuda()
    one = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_backproject(g, Q, s0, one)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.backproject_volume(og, Qn.astype(np.float64), s0=s0)
    assert_parity(one.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, "bp 600 views from s0=100")
    for cuts in ((100, 128, 384, 700), (100, 640, 700), (100, 256, 512, 640, 700)):
        part = torch.empty_like(one)
        for a, b in zip(cuts[:-1], cuts[1:]):
            ifdk_backproject(g, Q[a - s0:b - s0].contiguous(), a, part, accumulate=a > s0)
        assert torch.equal(part, one), cuts


def test_bp_band_not_covering_is_shape_error(torch_cuda):
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, IfdkError, ifdk_backproject

    spec = _spec(16, 64, 64, 32, 32, 32)
    g = Geometry.from_spec(spec)
    Q = torch.zeros((16, 10, 64), device="cuda")
    vol = torch.zeros((32, 32, 32), device="cuda")
    with pytest.raises(IfdkError) as e:
        ifdk_backproject(g, Q, 0, vol, v0=27)
    assert e.value.status == 3


def test_bp_zero_views(torch_cuda):
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject

    spec = _spec(16, 64, 64, 32, 32, 32)
    g = Geometry.from_spec(spec)
    vol = torch.ones((32, 32, 32), device="cuda")
    ifdk_backproject(g, torch.zeros((0, 64, 64), device="cuda"), 0, vol, accumulate=True)
    assert torch.all(vol == 1)
    ifdk_backproject(g, torch.zeros((0, 64, 64), device="cuda"), 0, vol)
    assert torch.all(vol == 0)


# ------------------------------------------------------------------------------- whole FDK
def test_reconstruct_config1(torch_cuda):
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct

    spec = synth.config(1)
    E = _phantom_E(spec)
    vol = torch.empty((64, 64, 64), device="cuda")
    ifdk_reconstruct(Geometry.from_spec(spec), torch.from_numpy(E).cuda(), vol)
    ref = oracle.reconstruct(oracle.OracleGeometry(**spec.geometry_args()), E)
    assert_parity(vol.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, "reconstruct config 1")


def test_reconstruct_noisy_stress_input(torch_cuda):
    """E + N(0, (0.01 max E)^2): roughens Q and stresses the coordinate numerics."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct

    spec = _spec(96, 128, 128, 96, 96, 96)
    E = _phantom_E(spec)
    E = synth.add_noise(E, 0.01 * float(E.max()), seed=1234)
    vol = torch.empty((96, 96, 96), device="cuda")
    ifdk_reconstruct(Geometry.from_spec(spec), torch.from_numpy(E).cuda(), vol)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.reconstruct(og, E, fft=True)
    assert_parity(vol.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, "reconstruct noisy")


@pytest.mark.parametrize("shape", [(48, 48, 48), (600, 24, 40)])  # (Nz, Ny, Nx)
def test_reconstruct_host_equals_device(torch_cuda, shape):
    """> one 256-view batch; Nz = 600 streams the last batch's volume to the host in slabs."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct, ifdk_reconstruct_host

    Nz, Ny, Nx = shape
    spec = _spec(300, 64, 64, Nx, Ny, Nz)
    g = Geometry.from_spec(spec)
    E = _phantom_E(spec)
    vol_d = torch.empty(shape, device="cuda")
    ifdk_reconstruct(g, torch.from_numpy(E).cuda(), vol_d)
    vol_h = np.empty(shape, np.float32)
    ifdk_reconstruct_host(g, E, vol_h)
    assert np.array_equal(vol_h, vol_d.cpu().numpy())
    ref = oracle.reconstruct(oracle.OracleGeometry(**spec.geometry_args()), E, fft=True)
    assert_parity(vol_h, ref, VOL_RMSE, VOL_MAX_REL, f"ifdk_reconstruct_host 300 views {shape}")


@pytest.mark.parametrize("shape,cuts", [((600, 24, 40), (0, 64, 300, 576, 600)),
                                        ((48, 48, 48), (0, 17, 48))])
def test_reconstruct_slab_host_zero_exchange(torch_cuda, shape, cuts):
    """Each slab reconstructed from its detector row band only (no exchange) equals
    the slab of the full reconstruction within fp32 rounding (rows pair up differently in the
    filter's transforms), including slabs not aligned to the 64-slice chunk and a 600-slice
    slab streamed back in pieces."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct, ifdk_reconstruct_slab_host

    Nz, Ny, Nx = shape
    spec = _spec(300, 64, 64, Nx, Ny, Nz)
    g = Geometry.from_spec(spec)
    E = _phantom_E(spec)
    vol_d = torch.empty(shape, device="cuda")
    ifdk_reconstruct(g, torch.from_numpy(E).cuda(), vol_d)
    full = vol_d.cpu().numpy()
    ref = oracle.reconstruct(oracle.OracleGeometry(**spec.geometry_args()), E, fft=True)
    got = np.empty(shape, np.float32)
    for a, b in zip(cuts[:-1], cuts[1:]):
        slab = np.empty((b - a, Ny, Nx), np.float32)
        ifdk_reconstruct_slab_host(g, E, a, slab)
        d = slab.astype(np.float64) - full[a:b]
        assert np.abs(d).max() <= 1e-5 * np.abs(full).max(), (a, b, np.abs(d).max())
        got[a:b] = slab
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL,
                  f"ifdk_reconstruct_slab_host 300 views {shape} slabs {cuts}")


def test_host_entry_points_config1_vs_oracle(torch_cuda):
    """Config 1 through every public end-to-end entry point, each against the oracle:
    ifdk_reconstruct_host, ifdk_reconstruct_slab_host (two slabs) and kslab_reconstruct_host."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct_host, ifdk_reconstruct_slab_host
    from paper_1909_02724_b200.dist import SlabPlan, kslab_reconstruct_host

    spec = synth.config(1)
    g = Geometry.from_spec(spec)
    E = _phantom_E(spec)
    ref = oracle.reconstruct(oracle.OracleGeometry(**spec.geometry_args()), E)
    vol_h = np.full((64, 64, 64), np.nan, np.float32)
    ifdk_reconstruct_host(g, E, vol_h)
    assert_parity(vol_h, ref, VOL_RMSE, VOL_MAX_REL, "config 1 ifdk_reconstruct_host")
    slabs = np.full((64, 64, 64), np.nan, np.float32)
    for a, b in ((0, 40), (40, 64)):
        part = np.empty((b - a, 64, 64), np.float32)
        ifdk_reconstruct_slab_host(g, E, a, part)
        slabs[a:b] = part
    assert_parity(slabs, ref, VOL_RMSE, VOL_MAX_REL, "config 1 ifdk_reconstruct_slab_host")
    raw_h = torch.from_numpy(E).pin_memory()
    vol_k = torch.full((64, 64, 64), float("nan")).pin_memory()
    vol_d = torch.empty((64, 64, 64), device="cuda")
    kslab_reconstruct_host(g, raw_h, vol_d, vol_k, SlabPlan(1, 64, 64), 0)
    torch.cuda.synchronize()
    assert_parity(vol_k.numpy(), ref, VOL_RMSE, VOL_MAX_REL, "config 1 kslab_reconstruct_host")


def test_synth_gpu_generator_matches_cpu(torch_cuda):
    torch = torch_cuda
    spec = synth.config(2)
    ell = synth.default_ellipsoids(spec)
    args = (spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell)
    out = torch.empty((3, 512, 512), device="cuda")
    synth.project_gpu(*args, 100, 3, 0, 512, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = synth.project(*args, 100, 3)
    assert np.max(np.abs(out.cpu().numpy() - ref)) <= 1e-5 * ref.max()


def test_kslab_driver_single_rank_equals_reconstruct(torch_cuda):
    """dist.kslab_reconstruct at world size 1 (pipelined rounds of 128-view blocks on three
    streams), its end-to-end host form, and the per-rank computation for world sizes 2 and 4
    (each rank's slab from the bands it would receive, round by round) are bitwise equal to
    ifdk_reconstruct."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, ifdk_filter, ifdk_reconstruct
    from paper_1909_02724_b200.dist import (SlabPlan, kslab_reconstruct, kslab_reconstruct_host,
                                            plan_exchange)

    spec = _spec(600, 128, 128, 96, 96, 320)  # 5 blocks: a short last block
    g = Geometry.from_spec(spec)
    raw = torch.from_numpy(_phantom_E(spec)).cuda()
    ref = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, raw, ref)
    plan1 = SlabPlan(1, spec.Nz, spec.Np)
    vol = torch.empty_like(ref)
    timings = {}
    kslab_reconstruct(g, raw, vol, plan1, 0, timings=timings)
    assert torch.equal(vol, ref)
    assert timings["rounds"] == 5 and timings["bp_ms"] > 0
    raw_h = raw.cpu().pin_memory()
    vol_h = torch.full(ref.shape, float("nan")).pin_memory()
    vol2 = torch.empty_like(ref)
    kslab_reconstruct_host(g, raw_h, vol2, vol_h, plan1, 0)
    torch.cuda.synchronize()
    assert torch.equal(vol_h, ref.cpu())
    oref = oracle.reconstruct(oracle.OracleGeometry(**spec.geometry_args()), raw_h.numpy(),
                              fft=True)
    assert_parity(vol_h.numpy(), oref, VOL_RMSE, VOL_MAX_REL, "kslab_reconstruct_host 600 views")
    Q = torch.empty_like(raw)
    ifdk_filter(g, raw, Q)
    for world in (2, 4):
        plan = SlabPlan(world, spec.Nz, spec.Np)
        for rank in range(world):
            k0, nk = plan.slab(rank)
            slab = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
            first = True
            for t in range(plan.n_rounds):
                ex = plan_exchange(g, plan, rank, t)
                for r in range(world):  # the bands rank r sends this rank in round t
                    s0, n = ex.views[r]
                    lo, hi = ex.recv[r]
                    if n == 0 or hi < lo:
                        continue
                    ifdk_backproject(g, Q[s0:s0 + n, lo:hi + 1].contiguous(), s0, slab, k0=k0,
                                     v0=lo, accumulate=not first)
                    first = False
            assert torch.equal(slab, ref[k0:k0 + nk]), (world, rank)


@pytest.mark.parametrize("seed", range(24))
def test_bp_random_geometries(torch_cuda, seed):
    """Random scanners (magnification, pitches, non-square detectors and volumes, odd sizes,
    view offsets, detectors smaller or larger than the shadow, 0.2 to 15 detector rows per
    slice) on a rough random Q: the patch bound never traps, every walk (QUAD / QUINT / PAIR /
    single, narrow / wide boxes) matches the oracle."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject

    rng = np.random.default_rng(1000 + seed)
    d = float(rng.uniform(300, 1500))
    spec = _spec(int(rng.integers(8, 41)), int(rng.integers(20, 91)), int(rng.integers(16, 81)),
                 int(rng.integers(8, 41)), int(rng.integers(8, 41)), int(rng.integers(8, 71)),
                 d=d, D=float(d * rng.uniform(1.2, 3.0)), det_mm=float(rng.uniform(100, 500)),
                 cube_mm=float(rng.uniform(50, 0.6 * d)))
    g = Geometry.from_spec(spec)
    s0 = int(rng.integers(-50, 50))
    n = spec.Np
    Q = rng.standard_normal((n, spec.Nv, spec.Nu)).astype(np.float32) * 100
    k0 = int(rng.integers(0, spec.Nz // 2))
    nk = int(rng.integers(1, spec.Nz - k0 + 1))
    vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
    ifdk_backproject(g, torch.from_numpy(Q).cuda(), s0, vol, k0=k0)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.backproject_volume(og, Q.astype(np.float64), s0=s0, k0=k0, nk=nk)
    assert_parity(vol.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, f"bp random geometry {seed}")


@pytest.mark.parametrize("family,walks,dims", [
    ("4-row TRIPLE", ("6", "9", "11"), (600, 96, 256, 48, 40, 128)),
    ("3-row TRIPLE", ("7", "10", "12"), (600, 96, 120, 48, 40, 128)),
])
def test_bp_tmem_walks_view_ranges(torch_cuda, auto_variant, family, walks, dims):
    """The TMEM-accumulator walks (9 / 10: one view per step; 11 / 12: two views per step, a
    one-view step where the first flush of the 128-view two-level sum falls on view 0 or at the
    last view) are bitwise the register walk (6 / 7) for view ranges that start off the
    128-view grid (s0 = 1, 37, 127, 128), have odd lengths and cross 256-view launch
    boundaries -- and for one and two views.  The 600-view result matches the oracle."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, set_bp_variant

    spec = _spec(*dims)
    g = Geometry.from_spec(spec)
    Qn = _oracle_Q32(spec, _phantom_E(spec))
    Q = torch.from_numpy(Qn).cuda()

    def run(w, s0, n):
        set_bp_variant(int(w))
        vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
        ifdk_backproject(g, Q[s0:s0 + n], s0, vol)
        torch.cuda.synchronize()
        return vol

    for s0, n in ((0, 600), (1, 300), (37, 219), (127, 2), (128, 1), (1, 1), (0, 2), (5, 131)):
        want = run(walks[0], s0, n)
        for w in walks[1:]:
            assert torch.equal(run(w, s0, n), want), (family, w, s0, n)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.backproject_volume(og, Qn.astype(np.float64), s0=0, v0=0, k0=0, nk=spec.Nz)
    assert_parity(run(walks[-1], 0, 600).cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL,
                  f"bp {family} TMEM two-view walk, 600 views")


@pytest.mark.parametrize("family,walks,dims", [
    ("4-row TRIPLE", ("11", "6", "3", "9"), (48, 96, 256, 48, 40, 256)),  # dv/dk 0.60-0.77
    ("3-row TRIPLE", ("12", "7", "8", "10"), (48, 96, 120, 48, 40, 256)),  # dv/dk 0.28-0.36
    ("PAIR", ("5", "4", "2"), (48, 96, 192, 48, 40, 256)),      # dv/dk in [0.45, 0.58]
    ("QUAD", ("13",), (48, 96, 256, 48, 40, 256)),              # masked partial chunks
    ("QUINT", ("14",), (48, 96, 120, 48, 40, 256)),             # masked partial chunks
    ("QUINT-HI", ("15",), (48, 96, 256, 48, 40, 256)),          # masked partial chunks
])
def test_bp_partial_chunks_far_into_the_chunk(torch_cuda, auto_variant, family, walks, dims):
    """Slab cuts deep inside a 64-slice chunk (k0 % 64 in {57, 59, 63}, ends 1, 3, 5 slices
    into the next chunk): the partial-chunk walks run the whole unrolled walk with masked
    slices whose floors lie outside the staged box; their shared loads are clamped into it
    (backproject.cu clamp_floor).  Every variant of the family is bitwise the
    whole-volume result, which matches the oracle.  Run under compute-sanitizer by
    tools/gpu_sanitize.sh."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, set_bp_variant

    spec = _spec(*dims)
    g = Geometry.from_spec(spec)
    Qn = _oracle_Q32(spec, _phantom_E(spec))
    Q = torch.from_numpy(Qn).cuda()

    def run(w, k0=0, nk=spec.Nz):
        set_bp_variant(int(w))
        lo = min(g.band_rows(k0, nk, s)[0] for s in range(spec.Np))
        hi = max(g.band_rows(k0, nk, s)[1] for s in range(spec.Np))
        vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
        ifdk_backproject(g, Q[:, lo:hi + 1].contiguous(), 0, vol, k0=k0, v0=lo)
        torch.cuda.synchronize()
        return vol

    whole = run(walks[0])
    for w in walks:
        for k0, k1 in ((57, 65), (59, 131), (63, 197), (121, 128), (64, 69), (185, 256)):
            assert torch.equal(run(w, k0, k1 - k0), whole[k0:k1]), (family, w, k0, k1)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.backproject_volume(og, Qn.astype(np.float64), s0=0, v0=0, k0=0, nk=spec.Nz)
    assert_parity(whole.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, f"bp {family} partial chunks")


@pytest.mark.parametrize("walk,dims", [
    (13, (600, 96, 256, 48, 40, 128)),  # QUAD: dv/dk in [0.60, 0.77] (configs 1-4)
    (14, (600, 96, 120, 48, 40, 128)),  # QUINT: dv/dk in [0.28, 0.36] (config 5)
    (15, (600, 96, 256, 48, 40, 128)),  # QUINT-HI: five-slice runs where 0.5 <= dv/dk < 1
])
def test_bp_quad_walk(torch_cuda, auto_variant, walk, dims):
    """QUAD / QUINT walks (13 / 14, the defaults where 0.5 <= dv/dk < 1 / dv/dk < 0.5): the
    automatic choice for their geometry; view ranges off the 128-view grid, odd lengths, one
    and two views and ranges crossing the 256-view launch boundary match the oracle; calls cut
    at multiples of the 128-view summation batch are bitwise one call; slab splits (the kernel
    walks partial chunks itself, masked write-back) are bitwise the whole volume."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, set_bp_variant

    spec = _spec(*dims)
    g = Geometry.from_spec(spec)
    Qn = _oracle_Q32(spec, _phantom_E(spec))
    Q = torch.from_numpy(Qn).cuda()
    og = oracle.OracleGeometry(**spec.geometry_args())

    def run(w, s0, n, k0=0, nk=spec.Nz, out=None, acc=False):
        set_bp_variant(int(w))
        vol = out if out is not None else torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
        ifdk_backproject(g, Q[s0:s0 + n], s0, vol, k0=k0, accumulate=acc)
        torch.cuda.synchronize()
        return vol

    default = run(walk, 0, 600)
    if walk != 15:  # the automatic choice for its geometry
        assert torch.equal(default, run(0, 0, 600))
    for s0, n in ((0, 600), (1, 300), (37, 219), (127, 2), (128, 1), (1, 1), (0, 2), (5, 131)):
        ref = oracle.backproject_volume(og, Qn[s0:s0 + n].astype(np.float64), s0=s0, v0=0, k0=0,
                                        nk=spec.Nz)
        assert_parity(run(walk, s0, n).cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL,
                      f"bp walk {walk} views {s0}..{s0 + n}")
    for cuts in ((0, 128, 384, 600), (0, 256, 600)):
        part = torch.empty_like(default)
        for a, b in zip(cuts[:-1], cuts[1:]):
            run(walk, a, b - a, out=part, acc=a > 0)
        assert torch.equal(part, default), cuts
    for a, b in ((0, 77), (77, 128), (3, 125), (64, 65), (57, 70)):
        assert torch.equal(run(walk, 0, 600, k0=a, nk=b - a), default[a:b]), (a, b)


def test_bp_many_detector_rows_per_slice(torch_cuda):
    """A scanner far outside the paper's regime: 14 mm voxels on 2.5 mm detector rows, 9-15 rows
    per slice (the single-slice walk).  Walked as fv0 + kk dv in fp32 the row position carried
    ulp(32 x 15) ~ 3e-5 px and this rough input reached relRMSE 1.2e-5; with dv split into
    whole rows + an fp32 fraction (ThreadInv.dvi / dvf) it matches the oracle."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject

    spec = _spec(23, 25, 78, 30, 38, 36, d=1253.3914983674254, D=3110.672396103071,
                 det_mm=195.808226584807, cube_mm=417.816532128783)
    g = Geometry.from_spec(spec)
    rng = np.random.default_rng(7)
    Q = rng.standard_normal((spec.Np, spec.Nv, spec.Nu)).astype(np.float32) * 100
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_backproject(g, torch.from_numpy(Q).cuda(), 0, vol)
    og = oracle.OracleGeometry(**spec.geometry_args())
    ref = oracle.backproject_volume(og, Q.astype(np.float64), s0=0, k0=0, nk=spec.Nz)
    assert_parity(vol.cpu().numpy(), ref, VOL_RMSE, VOL_MAX_REL, "bp 9-15 detector rows per slice")
