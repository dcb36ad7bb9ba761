"""A/B of bitwise-equal BP walks on one GPU (development aid, not the bench contract).

    python tools/ab_walk.py CONFIG WALK_A,WALK_B[,...] [n_views]

Times one n_views launch (default 256) of each walk over the whole volume (config 5: k-slab 0
of 8) with CUDA events and checks every volume is bitwise equal to the first walk's.  A walk
written W:R also sets the CTA raster band to R tile columns."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_backproject, ifdk_filter, set_bp_variant  # noqa: E402


def main(cfg, walks, n=256, reps=3):
    spec = synth.config(cfg)
    g = Geometry.from_spec(spec)
    nk = spec.Nz // 8 if cfg == 5 else spec.Nz
    E = torch.empty((n, spec.Nv, spec.Nu), device="cuda")
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                      synth.default_ellipsoids(spec), 0, n, 0, spec.Nv, E.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
    ifdk_filter(g, E, E)
    vols = {}
    for w in walks:
        wk, _, ra = str(w).partition(":")
        set_bp_variant(int(wk), int(ra) if ra else 0)
        vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
        ifdk_backproject(g, E, 0, vol)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            a.record()
            ifdk_backproject(g, E, 0, vol)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        t = min(ts)
        print(f"config {cfg} walk {w}: {t * 1e3:.1f} ms = {spec.Nx * spec.Ny * nk * n / t / 2**30:.1f} GUPS",
              flush=True)
        vols[w] = vol.cpu()
        del vol
    set_bp_variant(0, 0)
    for w in walks[1:]:
        eq = torch.equal(vols[walks[0]], vols[w])
        d = (vols[walks[0]] - vols[w]).abs().max().item()
        print(f"config {cfg} walks {walks[0]} vs {w}: bitwise equal {eq}, max |d| {d:.3e}",
              flush=True)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]), a[1].split(","), int(a[2]) if len(a) > 2 else 256)
