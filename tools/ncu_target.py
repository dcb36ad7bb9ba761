"""One filter launch + one BP launch on a config's first views (ncu capture target)."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_backproject, ifdk_filter  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
nk = int(sys.argv[3]) if len(sys.argv) > 3 else None
if len(sys.argv) > 4:  # BP walk (ifdk_set_bp_variant; bitwise-equal variants only)
    from paper_1909_02724_b200 import set_bp_variant

    set_bp_variant(int(sys.argv[4]))
spec = synth.config(cfg)
g = Geometry.from_spec(spec)
E = torch.empty((n, spec.Nv, spec.Nu), device="cuda")
synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                  synth.default_ellipsoids(spec), 0, n, 0, spec.Nv, E.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
Q = torch.empty_like(E)
nk = nk or spec.Nz
k0 = (spec.Nz - nk) // 2 // 64 * 64
vol = torch.empty((nk, spec.Ny, spec.Nx), device="cuda")
ifdk_filter(g, E, Q)
ifdk_backproject(g, Q, 0, vol, k0=k0)
torch.cuda.synchronize()
print("done", float(vol.abs().max()))
