"""Virtual ranks on one GPU for the fused projection split and the R x C grid (SURVEY 8(f)
row 2): every rank's back-projection adds its 128-view partial sums straight
into the owner's slab (ifdk_backproject_reduce, red.global.add) -- no partial volume, no
reduce-scatter.

* projection split (R = 1, C = P) for P = 1, 2, 4, 8: ranks run one after another;
* R x C grids (2x2, 4x2, 2x4, 1x3, 3x1): inside a column the k-slab pipeline with the fused
  band exchange (PeerExchange.local, wait / signal kernels), across a row the fused reduce into
  the row's chunk-aligned sub-slabs (grid.sub_bounds); every rank on its own three streams, all
  enqueued before any completes.

Each assembled volume must equal ifdk_reconstruct to fp32 summation order (max|d| <= 1e-5
max|V|; the atomic adds' order is not fixed) and a voxel sample must match the fp64 oracle.
Prints one line per case; exit 1 on a mismatch.  Used by tests/test_gpu_dist.py."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_reconstruct  # noqa: E402
from paper_1909_02724_b200.dist import (GridPlan, PeerExchange, ReduceSlabs,  # noqa: E402
                                        SlabPlan, exchanges, hybrid_reconstruct,
                                        projection_split_fused)
from parity_util import VOL_MAX_REL, VOL_RMSE, metrics  # noqa: E402
from virtual_ranks_check import _new_stream, watchdog  # noqa: E402


def main():
    torch.cuda.set_device(0)
    spec = synth.ConfigSpec("grid check", 600, 128, 128, 96, 96, 320)
    g = Geometry.from_spec(spec)
    raw_all = torch.empty((spec.Np, spec.Nv, spec.Nu), device="cuda")
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                      synth.default_ellipsoids(spec), 0, spec.Np, 0, spec.Nv, raw_all.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
    ref = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, raw_all, ref)
    torch.cuda.synchronize()
    vmax = float(ref.abs().max())
    rng = np.random.default_rng(20261017)
    ijk = np.stack([rng.integers(0, spec.Nx, 4096), rng.integers(0, spec.Ny, 4096),
                    rng.integers(0, spec.Nz, 4096)], 1).astype(np.int32)
    og = oracle.OracleGeometry(**spec.geometry_args())
    want = oracle.backproject(og, oracle.filter_fft(og, raw_all.cpu().numpy()), ijk)
    idx = torch.from_numpy(ijk.astype(np.int64)).cuda()
    bad = 0

    def check(what, vol):
        nonlocal bad
        err = float((vol - ref).abs().max()) / vmax
        r, m = metrics(vol[idx[:, 2], idx[:, 1], idx[:, 0]].cpu().numpy(), want)
        ok = err <= 1e-5 and r <= VOL_RMSE and m <= VOL_MAX_REL
        bad += not ok
        print(f"FUSED {what}: max|d|/max|V| vs one GPU {err:.2e}; oracle relRMSE {r:.2e} "
              f"max {m:.2e} {'OK' if ok else 'MISMATCH'}", flush=True)

    # projection split, P ranks one after another (no pipeline, no waits)
    for P in (1, 2, 4, 8):
        plan = SlabPlan(P, spec.Nz, spec.Np)
        slabs = ReduceSlabs.local(P, g, plan.k_bounds)
        for r in range(P):
            slabs[r].slab().zero_()
        for r in range(P):
            mine = [raw_all[s0:s0 + n] for s0, n in plan.local_views(r)]
            raw = torch.cat(mine) if mine else raw_all[:0]
            projection_split_fused(g, raw, plan.local_views(r), slabs[r], zero=False, sync=False)
        torch.cuda.synchronize()
        check(f"projection split P={P} (R=1, C={P})", torch.cat([slabs[h].slab() for h in range(P)]))
        slabs[0].close()

    # R x C grids: column pipelines (fused band exchange) + fused row reduce, all concurrent
    streams = [_new_stream() for _ in range(3 * 8)]
    # --no-wait: only grids without a band exchange (R = 1): the exchange's spinning wait kernels
    # need their peers' kernels to run concurrently, which compute-sanitizer does not allow
    grids = ((1, 3),) if "--no-wait" in sys.argv else ((2, 2), (4, 2), (2, 4), (1, 3), (3, 1))
    for R, C in grids:
        grid = GridPlan(R, C, spec.Nz, spec.Np)
        rows = [ReduceSlabs.local(C, g, grid.sub_bounds(r)) for r in range(R)]
        cols = []
        for c in range(C):
            plan = grid.column_plan(c)
            rmax = [max(sum(e.recv_sizes) for e in exchanges(g, plan, h)) for h in range(R)]
            pe = PeerExchange.local(R, rmax) if R > 1 else [None]
            for x in pe:
                if x is not None:
                    x.timeout_ms = 120000
            cols.append(pe)
        raws = {}
        for rank in range(R * C):
            r, c = grid.coords(rank)
            mine = [raw_all[s0:s0 + n] for s0, n in grid.column_plan(c).local_views(r)]
            raws[rank] = torch.cat(mine) if mine else raw_all[:0]
            rows[r][c].slab().zero_()
        torch.cuda.synchronize()
        for rank in range(R * C):
            r, c = grid.coords(rank)
            st = tuple(streams[3 * rank:3 * rank + 3])
            with torch.cuda.stream(st[2]):
                hybrid_reconstruct(g, raws[rank], None, grid, rank, None, None,
                                   peer=cols[c][r], slabs=rows[r][c], streams=st)
        watchdog([p for p in cols[0] if p is not None] or [None], R if R > 1 else 0,
                 f"grid {R}x{C}", [streams[3 * rank + 2] for rank in range(R * C)])
        vol = torch.cat([rows[r][c].slab() for r in range(R) for c in range(C)])
        check(f"R x C grid {R}x{C}", vol)
        for r in range(R):
            rows[r][0].close()
        for pe in cols:
            if pe[0] is not None:
                pe[0].close()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
