"""BP throughput on a k-slab (what one rank of the k-slab split computes): config, views, k0, nk."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_backproject, ifdk_filter  # noqa: E402

cfg, n, k0, nk = (int(a) for a in sys.argv[1:5])
spec = synth.config(cfg)
g = Geometry.from_spec(spec)
lo = min(g.band_rows(k0, nk, s)[0] for s in range(n))
hi = max(g.band_rows(k0, nk, s)[1] for s in range(n))
E = torch.empty((n, hi - lo + 1, spec.Nu), device="cuda")
synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                  synth.default_ellipsoids(spec), 0, n, lo, hi - lo + 1, E.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
Q = torch.empty_like(E)
ifdk_filter(g, E, Q, v0=lo)
vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
ifdk_backproject(g, Q, 0, vol, k0=k0, v0=lo)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    a.record()
    ifdk_backproject(g, Q, 0, vol, k0=k0, v0=lo)
    b.record()
    b.synchronize()
    t = a.elapsed_time(b) / 1e3
    print(f"config {cfg} slab k {k0}..{k0 + nk - 1}, {n} views, band {hi - lo + 1} rows: "
          f"BP {t * 1e3:.1f} ms = {spec.Nx * spec.Ny * nk * n / t / 2**30:.1f} GUPS", flush=True)
