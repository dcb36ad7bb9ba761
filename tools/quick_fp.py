"""Quick forward-projector / SART timing on one GPU (development aid, not the bench contract)."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1909_02724_b200 import SART, Geometry, ifdk_fill, ifdk_forward_project  # noqa: E402


def run(cfg, n_views=None, reps=2, sirt=False):
    spec = synth.config(cfg)
    n = spec.Np if n_views is None else n_views
    g = Geometry.from_spec(spec)
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_fill(vol, 1.0)
    proj = torch.empty((n, spec.Nv, spec.Nu), device="cuda")
    ifdk_forward_project(g, vol, 0, proj)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ups = spec.Nx * spec.Ny * spec.Nz * n
    for _ in range(reps):
        ev[0].record()
        ifdk_forward_project(g, vol, 0, proj)
        ev[1].record()
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1]) / 1e3
        print(f"config {cfg} views {n}: FP {t*1e3:.1f} ms = {ups/t/2**30:.1f} GUPS", flush=True)
    if sirt:
        st = SART(g, proj)
        x = torch.empty_like(vol)
        ifdk_fill(x, 0.0)
        st.iterate(x, 1)
        for _ in range(reps):
            ev[0].record()
            st.iterate(x, 1)
            ev[1].record()
            torch.cuda.synchronize()
            t = ev[0].elapsed_time(ev[1]) / 1e3
            print(f"config {cfg} views {n}: SIRT iteration {t*1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        c, _, nv = a.partition(":")
        run(int(c), int(nv) if nv else None, sirt=c in ("1", "2"))
