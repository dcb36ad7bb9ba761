"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The GPU reconstructs the whole config through the C ABI (ifdk_reconstruct: 256-view batches
of ifdk_filter + ifdk_backproject, exactly as in bench.py).  The oracle then recomputes a
deterministic voxel sample one voxel at a time (seed 20261017): random (i, j) on slices near
the central plane and random (i, j) on slices at the bottom of the volume.  Each sample lies
in a contiguous detector row band per view, so the oracle filters only those rows (fp64 FFT
form, pinned to the direct sum by test_oracle_pins) of every view and back-projects the
sampled voxels over all views (Alg. alg:bp).  Config 5 (4096^3, 256 GiB) does not fit one GPU;
its k-slab 0 (what rank 0 of 8 owns) is reconstructed from the row band that slab needs,
which is the per-rank computation of the k-slab split."""
import numpy as np
import pytest

import oracle
import synth
from parity_util import VOL_MAX_REL, VOL_RMSE, assert_parity

pytestmark = pytest.mark.gpu
SEED = 20261017


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _sample(spec, k_ranges, n_per, rng):
    parts = []
    for (ka, kb), n in zip(k_ranges, n_per):
        parts.append(np.stack([rng.integers(0, spec.Nx, n), rng.integers(0, spec.Ny, n),
                               rng.integers(ka, kb, n)], 1))
    return np.concatenate(parts).astype(np.int32)


def _band(gp, spec, ijk):
    ks = ijk[:, 2]
    k0, k1 = int(ks.min()), int(ks.max())
    lo, hi = 1 << 30, -1
    for s in range(spec.Np):
        a, b = gp.band_rows(k0, k1 - k0 + 1, s)
        lo, hi = min(lo, a), max(hi, b)
    return lo, hi


def _oracle_on_sample(spec, E_band, v0, ijk):
    og = oracle.OracleGeometry(**spec.geometry_args())
    Q = oracle.filter_fft(og, E_band, v0=v0)
    return oracle.backproject(og, Q, ijk, s0=0, v0=v0)


def _gen_raw(torch, spec, s0, n):
    raw = torch.empty((n, spec.Nv, spec.Nu), device="cuda")
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                      synth.default_ellipsoids(spec), s0, n, 0, spec.Nv, raw.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
    return raw


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_full_config_sampled_parity(torch_cuda, cfg):
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct

    spec = synth.config(cfg)
    g = Geometry.from_spec(spec)
    raw = _gen_raw(torch, spec, 0, spec.Np)
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, raw, vol)
    torch.cuda.synchronize()
    rng = np.random.default_rng(SEED)
    cz = spec.Nz // 2
    samples = {
        "central": _sample(spec, [(cz - 24, cz + 24)], [1 << 14], rng),
        # low slices that still cut the phantom (its z half-extent is 0.9 x 0.9 x 90 mm)
        "low": _sample(spec, [(spec.Nz // 10, spec.Nz // 10 + 12)], [1 << 13], rng),
    }
    for name, ijk in samples.items():
        lo, hi = _band(g, spec, ijk)
        E_band = raw[:, lo:hi + 1, :].cpu().numpy()
        ref = _oracle_on_sample(spec, E_band, lo, ijk)
        idx = torch.from_numpy(ijk.astype(np.int64)).cuda()
        got = vol[idx[:, 2], idx[:, 1], idx[:, 0]].cpu().numpy()
        assert np.abs(ref).max() > 0.05, f"{name} sample misses the phantom"
        assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, f"config {cfg} {name} sample")


def test_config5_slab0_sampled_parity(torch_cuda):
    """Config 5, k-slab 0 of 8 (512 slices): the views are filtered in 256-view batches and
    the slab is back-projected from the row band it needs, as one rank of the k-slab split."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, ifdk_filter
    from paper_1909_02724_b200.dist import SlabPlan, band_union

    spec = synth.config(5)
    g = Geometry.from_spec(spec)
    plan = SlabPlan(8, spec.Nz, spec.Np)
    k0, nk = plan.slab(0)
    vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
    batch = 256
    Q = torch.empty((batch, spec.Nv, spec.Nu), device="cuda")
    rng = np.random.default_rng(SEED)
    ijk = _sample(spec, [(k0 + nk - 16, k0 + nk - 8)], [1 << 13], rng)  # cuts the phantom
    lo_s, hi_s = _band(g, spec, ijk)
    E_band = np.empty((spec.Np, hi_s - lo_s + 1, spec.Nu), np.float32)
    for b0 in range(0, spec.Np, batch):
        raw = _gen_raw(torch, spec, b0, batch)
        E_band[b0:b0 + batch] = raw[:, lo_s:hi_s + 1, :].cpu().numpy()
        ifdk_filter(g, raw, Q)
        lo, hi = band_union(g, k0, nk, b0, batch)
        ifdk_backproject(g, Q[:, lo:hi + 1].contiguous(), b0, vol, k0=k0, v0=lo,
                         accumulate=b0 > 0)
        del raw
    torch.cuda.synchronize()
    ref = _oracle_on_sample(spec, E_band, lo_s, ijk)
    idx = torch.from_numpy(ijk.astype(np.int64)).cuda()
    got = vol[idx[:, 2] - k0, idx[:, 1], idx[:, 0]].cpu().numpy()
    assert np.abs(ref).max() > 0.05, "sample misses the phantom"
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, "config 5 slab 0 sample")
