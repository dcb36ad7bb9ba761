"""Virtual ranks on one GPU: the fused k-slab exchange of P = 2, 4, 8 ranks in ONE process --
the production PeerExchange layout (destination-relative band offsets, two receive areas per
rank, landed / freed signal words) driven by the real ifdk_filter_scatter (completion flags),
ifdk_wait and ifdk_signal kernels, every rank's pipeline on its own three streams.  Every
slab must be bitwise the single-GPU ifdk_reconstruct result, and a voxel sample matches the
fp64 oracle.  Prints one line per case; exit 1 on a mismatch.  Used by
tests/test_gpu_dist.py::test_virtual_ranks_fused_exchange.

All ranks' work is enqueued before any of it completes (a rank's wait kernels spin on the
GPU until its peers' scatters land), so every stream needs its own hardware queue:
CUDA_DEVICE_MAX_CONNECTIONS is raised before CUDA starts and the streams are created
directly (torch's stream pool could hand two ranks the same stream)."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_reconstruct  # noqa: E402
from paper_1909_02724_b200.dist import (PeerExchange, SlabPlan, exchanges,  # noqa: E402
                                        kslab_reconstruct, kslab_reconstruct_host)
from parity_util import VOL_MAX_REL, VOL_RMSE, metrics  # noqa: E402


def _new_stream():
    from cuda.bindings import runtime as cudart

    err, s = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
    assert int(err) == 0, err
    return torch.cuda.ExternalStream(int(s))


def watchdog(peers, P, what, joins, limit_s=90.0):
    """Wait for the enqueued pipelines (each rank joined into its stream in `joins`); if they
    do not finish in limit_s, print every rank's signal words (read through a side stream
    while the pipelines spin) and exit."""
    import time

    evs = []
    for st in joins:
        e = torch.cuda.Event()
        e.record(st)
        evs.append(e)
    side = _new_stream()
    t0 = time.time()
    print(f"enqueued {what}", flush=True)
    while not all(e.query() for e in evs):
        if time.time() - t0 > limit_s:
            from paper_1909_02724_b200.ifdk import as_tensor

            with torch.cuda.stream(side):
                for h in range(P):
                    w = as_tensor(peers[0].bases[h], (256,), "uint32").to("cpu", non_blocking=True)
                    side.synchronize()
                    w = w.tolist()
                    print(f"STUCK {what}: rank {h} landed={w[:P]} freed={w[64:64 + P]} "
                          f"ticket={w[128]}", flush=True)
            os._exit(3)
        time.sleep(0.05)
    print(f"joined {what} after {time.time() - t0:.2f} s", flush=True)
    torch.cuda.synchronize()
    print(f"synchronized {what}", flush=True)


def main():
    torch.cuda.set_device(0)
    spec = synth.ConfigSpec("virtual ranks", 600, 128, 128, 96, 96, 320)
    g = Geometry.from_spec(spec)
    raw_all = torch.empty((spec.Np, spec.Nv, spec.Nu), device="cuda")
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                      synth.default_ellipsoids(spec), 0, spec.Np, 0, spec.Nv, raw_all.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
    ref = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, raw_all, ref)
    torch.cuda.synchronize()
    streams = [_new_stream() for _ in range(3 * 8)]
    bad = 0
    for P, host in ((2, False), (4, False), (8, False), (2, True), (3, True)):
        plan = SlabPlan(P, spec.Nz, spec.Np)
        rmax = [max(sum(e.recv_sizes) for e in exchanges(g, plan, h)) for h in range(P)]
        peers = PeerExchange.local(P, rmax)
        for pe in peers:
            pe.timeout_ms = 120000
        # every input and output first: nothing below may block the host or join a stream
        # that another rank's pipeline is still waiting on
        raws, vols, hosts = [], [], []
        for r in range(P):
            k0, nk = plan.slab(r)
            mine = [raw_all[s0:s0 + n] for s0, n in plan.local_views(r)]
            # at P = 8 ranks 5-7 own no 128-view block of the 600 views: an empty shard
            raws.append(torch.cat(mine) if mine else raw_all[:0])
            vols.append(torch.full((nk, spec.Ny, spec.Nx), float("nan"), device="cuda"))
            if host:
                raws[-1] = raws[-1].cpu().pin_memory()
                hosts.append(torch.full((nk, spec.Ny, spec.Nx), float("nan"), pin_memory=True))
        torch.cuda.synchronize()
        for r in range(P):
            st = tuple(streams[3 * r:3 * r + 3])
            with torch.cuda.stream(st[2]):  # each rank joins its own copy stream, not a shared one
                if host:
                    kslab_reconstruct_host(g, raws[r], vols[r], hosts[r], plan, r, peer=peers[r],
                                           streams=st)
                else:
                    kslab_reconstruct(g, raws[r], vols[r], plan, r, peer=peers[r], streams=st)
        watchdog(peers, P, f"P={P} host={host}", [streams[3 * r + 2] for r in range(P)])
        full = torch.cat(vols)
        ok = torch.equal(full, ref)
        if host:
            ok = ok and torch.equal(torch.cat(hosts), ref.cpu())
        bad += not ok
        print(f"VIRTUAL P={P} host={host} used={peers[0].kind} "
              f"bitwise={'OK' if ok else 'MISMATCH'}", flush=True)
        peers[0].close()
    # the assembled volume against the fp64 oracle on a voxel sample (every slab)
    rng = np.random.default_rng(20261017)
    ijk = np.stack([rng.integers(0, spec.Nx, 4096), rng.integers(0, spec.Ny, 4096),
                    rng.integers(0, spec.Nz, 4096)], 1).astype(np.int32)
    og = oracle.OracleGeometry(**spec.geometry_args())
    E = raw_all.cpu().numpy()
    want = oracle.backproject(og, oracle.filter_fft(og, E), ijk)
    idx = torch.from_numpy(ijk.astype(np.int64)).cuda()
    got = ref[idx[:, 2], idx[:, 1], idx[:, 0]].cpu().numpy()
    r, m = metrics(got, want)
    ok = r <= VOL_RMSE and m <= VOL_MAX_REL
    bad += not ok
    print(f"PARITY virtual ranks vs oracle: relRMSE {r:.3e}  max|d|/max|ref| {m:.3e}  "
          f"{'OK' if ok else 'MISMATCH'}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
