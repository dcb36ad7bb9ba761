"""Under torchrun (NCCL): the k-slab driver with each exchange (fused filter + band scatter
into CUDA-IPC peer memory with device-side signals, and the NCCL all-to-all) equals
ifdk_reconstruct bitwise, and each rank's slab matches the fp64 oracle on a voxel sample.
Prints one line per exchange; exit code 1 on a mismatch.  Used by tests/test_gpu_dist.py.

KSLAB_SAME_GPU=1: every rank on cuda:0 with a gloo process group (NCCL refuses two ranks on
one GPU) and only the fused exchange -- real cross-process IPC mappings and signals between
time-sliced contexts, the multi-process path a one-GPU box can run."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from parity_util import VOL_MAX_REL, VOL_RMSE, metrics  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_reconstruct  # noqa: E402
from paper_1909_02724_b200.dist import (ReduceSlabs, SlabPlan, kslab_reconstruct,  # noqa: E402
                                        kslab_reconstruct_host, projection_split_fused,
                                        projection_split_reconstruct)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    same_gpu = os.environ.get("KSLAB_SAME_GPU") == "1"
    torch.cuda.set_device(0 if same_gpu else int(os.environ.get("LOCAL_RANK", 0)))
    if same_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl",
                                device_id=torch.device("cuda", torch.cuda.current_device()))
    spec = synth.ConfigSpec("kslab check", 600, 128, 128, 96, 96, 320)
    g = Geometry.from_spec(spec)
    ell = synth.default_ellipsoids(spec)
    raw_all = torch.empty((spec.Np, spec.Nv, spec.Nu), device="cuda")
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, 0,
                      spec.Np, 0, spec.Nv, raw_all.data_ptr(), torch.cuda.current_stream().cuda_stream)
    ref = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, raw_all, ref)
    plan = SlabPlan(world, spec.Nz, spec.Np)
    k0, nk = plan.slab(rank)
    raw = torch.cat([raw_all[s0:s0 + n] for s0, n in plan.local_views(rank)])
    bad = 0
    # this rank's slab against the fp64 oracle on a voxel sample (both slab faces included)
    rng = np.random.default_rng(20261017 + rank)
    ks = np.concatenate([rng.integers(k0, k0 + nk, 1024), np.full(256, k0), np.full(256, k0 + nk - 1)])
    ijk = np.stack([rng.integers(0, spec.Nx, ks.size), rng.integers(0, spec.Ny, ks.size), ks],
                   1).astype(np.int32)
    og = oracle.OracleGeometry(**spec.geometry_args())
    want = oracle.backproject(og, oracle.filter_fft(og, raw_all.cpu().numpy()), ijk)
    idx = torch.from_numpy(ijk.astype(np.int64)).cuda()
    for exchange in (("p2p",) if same_gpu else ("auto", "nccl")):
        vol = torch.full((nk, spec.Ny, spec.Nx), float("nan"), device="cuda")
        tm = {}
        for _ in range(2):  # twice: the second call reuses the cached symmetric buffers
            kslab_reconstruct(g, raw, vol, plan, rank, timings=tm, force_exchange=True,
                              exchange=exchange)
        ok = torch.equal(vol, ref[k0:k0 + nk])
        r_, m_ = metrics(vol[idx[:, 2] - k0, idx[:, 1], idx[:, 0]].cpu().numpy(), want)
        ok_o = r_ <= VOL_RMSE and m_ <= VOL_MAX_REL
        bad += (not ok) + (not ok_o)
        print(f"KSLAB rank {rank}/{world} exchange={exchange} used={tm.get('exchange')} "
              f"bitwise={'OK' if ok else 'MISMATCH'} oracle relRMSE={r_:.2e} max={m_:.2e} "
              f"{'ORACLE-OK' if ok_o else 'ORACLE-MISMATCH'} wall={tm.get('wall_ms', 0):.1f} ms "
              f"delta={tm.get('delta') or 0:.2f}", flush=True)
    # end to end from pinned host memory (H2D one round ahead, D2H in sub-slabs)
    raw_h = raw.cpu().pin_memory()
    vol_h = torch.empty((nk, spec.Ny, spec.Nx), dtype=torch.float32, pin_memory=True)
    vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
    kslab_reconstruct_host(g, raw_h, vol, vol_h, plan, rank, force_exchange=True,
                           exchange="p2p" if same_gpu else "auto")
    torch.cuda.synchronize()
    ok = torch.equal(vol_h, ref[k0:k0 + nk].cpu())
    bad += not ok
    print(f"KSLAB-HOST rank {rank}/{world} bitwise={'OK' if ok else 'MISMATCH'}", flush=True)
    # projection split: partial volume of the own views + NCCL reduce-scatter of k-slabs
    if spec.Nz % world == 0 and not same_gpu:
        ps = torch.empty((spec.Nz // world, spec.Ny, spec.Nx), device="cuda")
        projection_split_reconstruct(g, raw, plan.local_views(rank), ps, world)
        r0 = rank * spec.Nz // world
        refp = ref[r0:r0 + spec.Nz // world]
        err = float((ps - refp).abs().max() / ref.abs().max())
        ok = err <= 1e-5
        bad += not ok
        print(f"PSPLIT rank {rank}/{world} max|d|/max|V|={err:.2e} {'OK' if ok else 'MISMATCH'}",
              flush=True)
    # fused projection split: every rank's partial sums added straight into the owners' slabs
    # (IPC-mapped: a peer's device memory), no partial volume, no reduce-scatter
    slabs = ReduceSlabs.create(None, rank, world, g, plan.k_bounds)
    own = projection_split_fused(g, raw, plan.local_views(rank), slabs)
    err = float((own - ref[k0:k0 + nk]).abs().max() / ref.abs().max())
    r_, m_ = metrics(own[idx[:, 2] - k0, idx[:, 1], idx[:, 0]].cpu().numpy(), want)
    ok = err <= 1e-5 and r_ <= VOL_RMSE and m_ <= VOL_MAX_REL
    bad += not ok
    print(f"PSFUSED rank {rank}/{world} max|d|/max|V|={err:.2e} oracle relRMSE={r_:.2e} "
          f"max={m_:.2e} {'OK' if ok else 'MISMATCH'}", flush=True)
    dist.barrier()
    slabs.close()
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
