"""Quick BP/filter timing on one GPU (development aid, not the bench contract)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_backproject, ifdk_filter  # noqa: E402


def run(cfg, n_views=None, reps=2):
    spec = synth.config(cfg)
    n = spec.Np if n_views is None else n_views
    g = Geometry.from_spec(spec)
    E = torch.empty((n, spec.Nv, spec.Nu), device="cuda")
    ell = synth.default_ellipsoids(spec)
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, 0, n, 0,
                      spec.Nv, E.data_ptr(), torch.cuda.current_stream().cuda_stream)
    Q = torch.empty_like(E)
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_filter(g, E, Q)
    ifdk_backproject(g, Q, 0, vol)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(reps):
        ev[0].record()
        ifdk_filter(g, E, Q)
        ev[1].record()
        ifdk_backproject(g, Q, 0, vol)
        ev[2].record()
        torch.cuda.synchronize()
        tf = ev[0].elapsed_time(ev[1]) / 1e3
        tb = ev[1].elapsed_time(ev[2]) / 1e3
        ups = spec.Nx * spec.Ny * spec.Nz * n
        print(f"config {cfg} views {n}: filter {tf*1e3:.2f} ms ({8*E.numel()/tf/1e9:.0f} GB/s), "
              f"BP {tb*1e3:.1f} ms = {ups/tb/2**30:.1f} GUPS", flush=True)
    del E, Q, vol
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for a in sys.argv[1:]:
        c, _, nv = a.partition(":")
        run(int(c), int(nv) if nv else None)
