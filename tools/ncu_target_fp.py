"""One forward-projector launch (ncu capture target): config 3 geometry, phantom volume."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_fill, ifdk_forward_project  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
spec = synth.config(cfg)
g = Geometry.from_spec(spec)
vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
ifdk_fill(vol, 1.0)
proj = torch.empty((n, spec.Nv, spec.Nu), device="cuda")
ifdk_forward_project(g, vol, 0, proj)
torch.cuda.synchronize()
print("done", float(proj.abs().max()))
