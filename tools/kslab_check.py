"""Under torchrun (NCCL): the k-slab driver with each exchange (fused filter + P2P band scatter
over symmetric memory, and the NCCL all-to-all) equals ifdk_reconstruct bitwise.  Prints one
line per exchange; exit code 1 on a mismatch.  Used by tests/test_gpu_dist.py."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_reconstruct  # noqa: E402
from paper_1909_02724_b200.dist import (SlabPlan, kslab_reconstruct,  # noqa: E402
                                        kslab_reconstruct_host, projection_split_reconstruct)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
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
    for exchange in ("auto", "nccl"):
        vol = torch.full((nk, spec.Ny, spec.Nx), float("nan"), device="cuda")
        tm = {}
        for _ in range(2):  # twice: the second call reuses the cached symmetric buffers
            kslab_reconstruct(g, raw, vol, plan, rank, timings=tm, force_exchange=True,
                              exchange=exchange)
        ok = torch.equal(vol, ref[k0:k0 + nk])
        bad += not ok
        print(f"KSLAB rank {rank}/{world} exchange={exchange} used={tm.get('exchange')} "
              f"bitwise={'OK' if ok else 'MISMATCH'} wall={tm.get('wall_ms', 0):.1f} ms", flush=True)
    # end to end from pinned host memory (H2D one round ahead, D2H in sub-slabs)
    raw_h = raw.cpu().pin_memory()
    vol_h = torch.empty((nk, spec.Ny, spec.Nx), dtype=torch.float32, pin_memory=True)
    vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
    kslab_reconstruct_host(g, raw_h, vol, vol_h, plan, rank, force_exchange=True)
    torch.cuda.synchronize()
    ok = torch.equal(vol_h, ref[k0:k0 + nk].cpu())
    bad += not ok
    print(f"KSLAB-HOST rank {rank}/{world} bitwise={'OK' if ok else 'MISMATCH'}", flush=True)
    # projection split: partial volume of the own views + NCCL reduce-scatter of k-slabs
    if spec.Nz % world == 0:
        ps = torch.empty((spec.Nz // world, spec.Ny, spec.Nx), device="cuda")
        projection_split_reconstruct(g, raw, plan.local_views(rank), ps, world)
        r0 = rank * spec.Nz // world
        refp = ref[r0:r0 + spec.Nz // world]
        err = float((ps - refp).abs().max() / ref.abs().max())
        ok = err <= 1e-5
        bad += not ok
        print(f"PSPLIT rank {rank}/{world} max|d|/max|V|={err:.2e} {'OK' if ok else 'MISMATCH'}",
              flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
