"""Where does end-to-end time go? PCIe bandwidths and ifdk_reconstruct_host phases (dev aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1909_02724_b200 import Geometry, ifdk_reconstruct, ifdk_reconstruct_host  # noqa: E402


def bw():
    n = 1 << 30  # 4 GiB of fp32
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in [("H2D", lambda: d.copy_(h, non_blocking=True)),
                     ("D2H", lambda: h.copy_(d, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(f"{name} 4 GiB pinned: {4 * 2**30 / dt / 1e9:.1f} GB/s", flush=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"bidirectional 2 x 4 GiB: {8 * 2**30 / dt / 1e9:.1f} GB/s total", flush=True)
    del h, d, h2, d2
    torch.cuda.empty_cache()


def e2e(cfg):
    spec = synth.config(cfg)
    g = Geometry.from_spec(spec)
    raw = torch.empty((spec.Np, spec.Nv, spec.Nu), device="cuda")
    ell = synth.default_ellipsoids(spec)
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, 0,
                      spec.Np, 0, spec.Nv, raw.data_ptr(), torch.cuda.current_stream().cuda_stream)
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    ifdk_reconstruct(g, raw, vol)
    torch.cuda.synchronize()
    t = time.perf_counter(); ifdk_reconstruct(g, raw, vol); torch.cuda.synchronize()
    dev_s = time.perf_counter() - t
    raw_h = torch.empty(raw.shape, dtype=torch.float32, pin_memory=True)
    raw_h.copy_(raw)
    vol_h = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
    del raw, vol
    torch.cuda.empty_cache()
    ifdk_reconstruct_host(g, raw_h, vol_h)
    for _ in range(2):
        t = time.perf_counter(); ifdk_reconstruct_host(g, raw_h, vol_h)
        host_s = time.perf_counter() - t
        print(f"config {cfg}: device reconstruct {dev_s:.3f} s, reconstruct_host {host_s:.3f} s",
              flush=True)


if __name__ == "__main__":
    bw()
    for a in sys.argv[1:]:
        e2e(int(a))
