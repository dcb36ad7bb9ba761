"""SURVEY 8(d)'s parity set at BASELINE.json's full sizes, in the launch configuration bench.py
times, against the fp64 oracle on the same generated fp32 projections.

- Config 2 (512^3): the FULL volume (Alg. alg:bp over every voxel; oracle filter in its FFT
  form, pinned to the direct sum by test_oracle_pins).
- Configs 3 and 4: a deterministic sample (seed 20261017) -- 2^20 random voxels, the 3
  central planes, both planes at every slab boundary of the P = 2/4/8 k-slab splits (the last
  slice of slab m-1 and the first of slab m) and the 8 corners.  Planes are row-sampled (whole
  i-rows at random j), as SURVEY 8(d)'s cost note allows.  Config 3 runs through the
  end-to-end host entry point ifdk_reconstruct_host (the bench's e2e call), config 4 through
  ifdk_reconstruct (the bench's device-resident step).
- Config 5 (4096^3, 256 GiB: one slab per rank at P = 8): all 8 k-slabs, one at a time,
  each back-projected as its rank does (k0, nk from SlabPlan) and sampled on both slab faces,
  plus the 8 corners of the volume.

The oracle side streams the views in batches: each batch's raw rows are copied to the host,
filtered by oracle.filter_fft and back-projected over the sampled voxels by
oracle.backproject(s0 = first view of the batch); the per-batch partial sums are added in fp64
in view order.  Metrics are relRMSE and max|d| / max|V| over the sample (north_star; max|V|
lies on the central planes).  The oracle work runs on a host thread so that it overlaps the
GPU work."""
import concurrent.futures as cf
import time

import numpy as np
import pytest

import oracle
import synth
from parity_util import VOL_MAX_REL, VOL_RMSE, assert_parity, filter_fft_threads, metrics

pytestmark = pytest.mark.gpu
SEED = 20261017
ORACLE_BATCH = 64  # views per oracle filter/BP batch (2 GiB of fp64 Q at config 4)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _gen_raw(torch, spec, s0, n, out=None):
    raw = torch.empty((n, spec.Nv, spec.Nu), device="cuda") if out is None else out
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                      synth.default_ellipsoids(spec), s0, n, 0, spec.Nv, raw.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
    return raw


def _rows_of_planes(rng, spec, ks, n_rows):
    """Whole i-rows at n_rows random j on each plane k of ks."""
    parts = []
    i = np.arange(spec.Nx)
    for k in ks:
        for j in rng.choice(spec.Ny, size=n_rows, replace=False):
            parts.append(np.stack([i, np.full_like(i, j), np.full_like(i, k)], 1))
    return np.concatenate(parts)


def _corners(spec):
    return np.array([[i, j, k] for k in (0, spec.Nz - 1) for j in (0, spec.Ny - 1)
                     for i in (0, spec.Nx - 1)])


def slab_boundaries(spec):
    """Every interior slab boundary of the P = 2/4/8 k-slab splits (SlabPlan's cuts)."""
    from paper_1909_02724_b200.dist import SlabPlan

    cuts = set()
    for P in (2, 4, 8):
        cuts.update(SlabPlan(P, spec.Nz, spec.Np).k_bounds[1:-1])
    return sorted(cuts)


def parity_sample(spec, n_random=1 << 20, central_rows=16, boundary_rows=8):
    """SURVEY 8(d)'s sample for configs 3-4: name -> (n, 3) int32 (i, j, k)."""
    rng = np.random.default_rng(SEED)
    cz = spec.Nz // 2
    bnd = slab_boundaries(spec) if boundary_rows else []
    groups = {
        "random": np.stack([rng.integers(0, spec.Nx, n_random), rng.integers(0, spec.Ny, n_random),
                            rng.integers(0, spec.Nz, n_random)], 1),
        "central planes": _rows_of_planes(rng, spec, (cz - 1, cz, cz + 1), central_rows),
        "slab-boundary planes": _rows_of_planes(
            rng, spec, [k for b in bnd for k in (b - 1, b)], boundary_rows) if bnd
        else np.zeros((0, 3), np.int64),
        "corners": _corners(spec),
    }
    return {k: v.astype(np.int32) for k, v in groups.items()}


class OracleSum:
    """The oracle over view batches for voxel groups that each need detector rows lo..hi:
    V[group] = sum over batches (view order) of oracle.backproject(filter_fft(E rows))."""

    def __init__(self, spec, groups):
        self.og = oracle.OracleGeometry(**spec.geometry_args())
        self.groups = groups  # name -> (ijk, lo, hi)
        self.acc = {name: np.zeros(len(ijk)) for name, (ijk, _, _) in groups.items()}
        self.seconds = 0.0
        self.updates = 0

    def add(self, s0, E, v0):
        """E: [n][rows][Nu] fp32 raw views s0.., detector rows v0.. (covering every group)."""
        t = time.perf_counter()
        for name, (ijk, lo, hi) in self.groups.items():
            Q = filter_fft_threads(self.og, E[:, lo - v0:hi - v0 + 1], v0=lo)
            self.acc[name] += oracle.backproject(self.og, Q, ijk, s0=s0, v0=lo)
            self.updates += len(ijk) * E.shape[0]
        self.seconds += time.perf_counter() - t


class Background:
    """One host worker for the oracle, with a bounded queue (host memory)."""

    def __init__(self, depth=3):
        self.ex = cf.ThreadPoolExecutor(max_workers=1)
        self.pending = []
        self.depth = depth

    def submit(self, fn, *args):
        self.pending.append(self.ex.submit(fn, *args))
        while len(self.pending) > self.depth:
            self.pending.pop(0).result()

    def join(self):
        for f in self.pending:
            f.result()
        self.pending = []
        self.ex.shutdown()


def _gather(torch, vol, ijk, k0=0):
    idx = torch.from_numpy(ijk.astype(np.int64)).to(vol.device)
    return vol[idx[:, 2] - k0, idx[:, 1], idx[:, 0]].cpu().numpy()


def _report(spec, groups_got, groups_ref, what):
    got = np.concatenate([groups_got[n] for n in groups_ref])
    ref = np.concatenate([groups_ref[n] for n in groups_ref])
    vmax = float(np.abs(ref).max())
    assert vmax > 0.5, f"{what}: the sample misses the phantom (max|V| = {vmax})"
    for n in groups_ref:  # per-group lines, each against the sample's max|V|
        d = np.abs(groups_got[n].astype(np.float64) - groups_ref[n])
        r, _ = metrics(groups_got[n], groups_ref[n])
        print(f"PARITY {what} [{n}]: relRMSE {r:.3e}  max|d|/max|V| {d.max() / vmax:.3e}  "
              f"(n={len(d)})")
        assert d.max() <= VOL_MAX_REL * vmax, (n, d.max() / vmax)
    return assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, what)


# ------------------------------------------------------------------------------ config 2
@pytest.mark.slow
def test_config2_full_volume_parity(torch_cuda):
    """Config 2, all 2^27 voxels against the oracle (2^36 oracle updates, ~5 min on 16 cores)."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct

    spec = synth.config(2)
    g = Geometry.from_spec(spec)
    raw = _gen_raw(torch, spec, 0, spec.Np)
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, raw, vol)
    E = raw.cpu().numpy()
    got = vol.cpu().numpy()
    del raw, vol
    og = oracle.OracleGeometry(**spec.geometry_args())
    t = time.perf_counter()
    ref = oracle.backproject_volume(og, filter_fft_threads(og, E))
    dt = time.perf_counter() - t
    print(f"ORACLE config 2 full volume: {dt:.1f} s, {spec.updates / dt / 1e9:.3f} G updates/s "
          f"on {oracle.num_threads()} threads")
    assert np.abs(ref).max() > 0.5
    assert_parity(got, ref, VOL_RMSE, VOL_MAX_REL, "config 2 full volume")


# --------------------------------------------------------------------------- configs 3-4
def _oracle_full_rows(torch, spec, groups, E_of, bg):
    """Stream every view's full detector to the oracle (the random sample needs every row)."""
    osum = OracleSum(spec, {n: (ijk, 0, spec.Nv - 1) for n, ijk in groups.items()})
    for b0 in range(0, spec.Np, ORACLE_BATCH):
        n = min(ORACLE_BATCH, spec.Np - b0)
        bg.submit(osum.add, b0, E_of(b0, n), 0)
    return osum


def test_config3_parity_set_via_host_entry(torch_cuda):
    """Config 3 end to end from host memory (ifdk_reconstruct_host: H2D, filter, BP, D2H)."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct_host

    spec = synth.config(3)
    g = Geometry.from_spec(spec)
    raw_h = _gen_raw(torch, spec, 0, spec.Np).cpu()
    E = raw_h.numpy()
    groups = parity_sample(spec)
    bg = Background()
    osum = _oracle_full_rows(torch, spec, groups, lambda b0, n: E[b0:b0 + n], bg)
    vol_h = np.full((spec.Nz, spec.Ny, spec.Nx), np.nan, np.float32)
    ifdk_reconstruct_host(g, raw_h, vol_h)
    bg.join()
    got = {n: vol_h[ijk[:, 2], ijk[:, 1], ijk[:, 0]] for n, ijk in groups.items()}
    print(f"ORACLE config 3 sample: {osum.seconds:.1f} s, {osum.updates / osum.seconds / 1e9:.3f}"
          f" G updates/s")
    assert not np.isnan(vol_h).any()
    _report(spec, got, osum.acc, "config 3 parity set (ifdk_reconstruct_host)")


def test_config4_parity_set(torch_cuda):
    """Config 4 through ifdk_reconstruct (the device-resident FDK step bench.py times)."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct

    spec = synth.config(4)
    g = Geometry.from_spec(spec)
    raw = _gen_raw(torch, spec, 0, spec.Np)
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, raw, vol)
    groups = parity_sample(spec)
    got = {n: _gather(torch, vol, ijk) for n, ijk in groups.items()}
    del vol
    bg = Background()
    osum = _oracle_full_rows(torch, spec, groups, lambda b0, n: raw[b0:b0 + n].cpu().numpy(), bg)
    bg.join()
    del raw
    print(f"ORACLE config 4 sample: {osum.seconds:.1f} s, {osum.updates / osum.seconds / 1e9:.3f}"
          f" G updates/s")
    _report(spec, got, osum.acc, "config 4 parity set")


def test_config3_noisy_stress_input(torch_cuda):
    """SURVEY 8(d)'s stress input at full size: config 3 with E + N(0, (0.01 max E)^2) (seed 1234,
    counter-based, synth.add_noise), which roughens Q and amplifies coordinate error (c-N1);
    2^18 random voxels + the central planes against the oracle on the same noisy fp32 input."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_reconstruct

    spec = synth.config(3)
    g = Geometry.from_spec(spec)
    E = _gen_raw(torch, spec, 0, spec.Np).cpu().numpy()
    E = synth.add_noise(E, 0.01 * float(E.max()), seed=1234)
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, torch.from_numpy(E).cuda(), vol)
    groups = parity_sample(spec, n_random=1 << 18, boundary_rows=0)
    groups.pop("slab-boundary planes")
    got = {n: _gather(torch, vol, ijk) for n, ijk in groups.items()}
    del vol
    bg = Background()
    osum = _oracle_full_rows(torch, spec, groups, lambda b0, n: E[b0:b0 + n], bg)
    bg.join()
    _report(spec, got, osum.acc, "config 3 noisy stress input")


# ------------------------------------------------------------------------------ config 5
def test_config5_all_slabs_face_parity(torch_cuda):
    """Config 5: every k-slab of the P = 8 split, back-projected one at a time from the
    filtered views (the per-rank computation of the k-slab split), sampled on both faces.

    Filtered views stay resident (64 GiB) and each slab (32 GiB) is back-projected from them in
    256-view launches, as a rank does.  The oracle filters only the detector rows the face
    samples need (union of ifdk_band_rows over the views; the oracle raises if a needed tap is
    outside the rows it was given)."""
    torch = torch_cuda
    from paper_1909_02724_b200 import Geometry, ifdk_backproject, ifdk_filter
    from paper_1909_02724_b200.dist import SlabPlan

    spec = synth.config(5)
    g = Geometry.from_spec(spec)
    plan = SlabPlan(8, spec.Nz, spec.Np)
    rng = np.random.default_rng(SEED)
    n_face = 1 << 14
    faces = {}  # k -> ijk
    for r in range(8):
        k0, nk = plan.slab(r)
        for k in (k0, k0 + nk - 1):
            faces[k] = np.stack([rng.integers(0, spec.Nx, n_face), rng.integers(0, spec.Ny, n_face),
                                 np.full(n_face, k)], 1).astype(np.int32)
    corners = _corners(spec).astype(np.int32)
    faces[0] = np.concatenate([faces[0], corners[corners[:, 2] == 0]])
    faces[spec.Nz - 1] = np.concatenate([faces[spec.Nz - 1], corners[corners[:, 2] > 0]])
    # faces that touch (the last slice of slab r-1, the first of slab r) share one oracle
    # group: one filter pass over the union of their row bands
    groups, where = {}, {}
    for k in sorted(faces):
        key = f"boundary {((k + 1) // plan.slab(0)[1]) * plan.slab(0)[1]}"
        ijk = faces[k]
        if key in groups:
            prev = groups[key][0]
            where[k] = (key, len(prev), len(prev) + len(ijk))
            ijk = np.concatenate([prev, ijk])
        else:
            where[k] = (key, 0, len(ijk))
        groups[key] = (ijk, 0, 0)
    for key, (ijk, _, _) in groups.items():
        lo, hi = 1 << 30, -1
        ka, kb = int(ijk[:, 2].min()), int(ijk[:, 2].max())
        for s in range(spec.Np):
            a, b = g.band_rows(ka, kb - ka + 1, s)
            lo, hi = min(lo, a), max(hi, b)
        groups[key] = (ijk, lo, hi)
    v_lo = min(lo for _, lo, _ in groups.values())
    v_hi = max(hi for _, _, hi in groups.values())
    rows = np.zeros(spec.Nv, bool)
    for _, lo, hi in groups.values():
        rows[lo:hi + 1] = True
    osum = OracleSum(spec, groups)
    bg = Background(depth=2)

    batch = 256
    Q = torch.empty((spec.Np, spec.Nv, spec.Nu), device="cuda")  # 64 GiB
    raw = torch.empty((batch, spec.Nv, spec.Nu), device="cuda")
    sel = torch.from_numpy(np.nonzero(rows)[0]).cuda()
    for b0 in range(0, spec.Np, batch):
        _gen_raw(torch, spec, b0, batch, out=raw)
        ifdk_filter(g, raw, Q[b0:b0 + batch])
        # only the rows the oracle needs go to the host; unneeded rows are left as zero
        E = np.zeros((batch, v_hi - v_lo + 1, spec.Nu), np.float32)
        E[:, rows[v_lo:v_hi + 1]] = raw.index_select(1, sel).cpu().numpy()
        bg.submit(osum.add, b0, E, v_lo)
    del raw
    vol = torch.empty((plan.slab(0)[1], spec.Ny, spec.Nx), device="cuda")  # 32 GiB
    got = {}
    for r in range(8):
        k0, nk = plan.slab(r)
        for s0 in range(0, spec.Np, batch):
            ifdk_backproject(g, Q[s0:s0 + batch], s0, vol, k0=k0, v0=0, accumulate=s0 > 0)
        for k in (k0, k0 + nk - 1):
            got[k] = _gather(torch, vol, faces[k], k0=k0)
    del vol, Q
    bg.join()
    print(f"ORACLE config 5 faces: {osum.seconds:.1f} s, {osum.updates / osum.seconds / 1e9:.3f}"
          f" G updates/s")
    ref = {k: osum.acc[key][a:b] for k, (key, a, b) in where.items()}
    vmax = max(float(np.abs(v).max()) for v in ref.values())
    for r in range(8):
        k0, nk = plan.slab(r)
        names = [k0, k0 + nk - 1]
        d = np.concatenate([got[n].astype(np.float64) - ref[n] for n in names])
        rr, _ = metrics(np.concatenate([got[n] for n in names]),
                        np.concatenate([ref[n] for n in names]))
        print(f"PARITY config 5 slab {r} (k {k0}..{k0 + nk - 1}) faces: relRMSE {rr:.3e}  "
              f"max|d|/max|V| {np.abs(d).max() / vmax:.3e}  (n={len(d)})")
        assert np.abs(d).max() <= VOL_MAX_REL * vmax, (r, np.abs(d).max() / vmax)
    assert vmax > 0.05
    assert_parity(np.concatenate([got[n] for n in ref]), np.concatenate([ref[n] for n in ref]),
                  VOL_RMSE, VOL_MAX_REL, "config 5 all slab faces")
