"""Production BP vs the paper-style baselines on B200: GUPS of each kernel
and the error of each whole path (GPU filter + BP) against the fp64 oracle on the config-3
central-plane sample.  Writes gpurun_out/baselines.json (dev tool behind DESIGN.md)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1909_02724_b200 import (Geometry, ifdk_backproject, ifdk_backproject_alg2,  # noqa: E402
                                   ifdk_backproject_alg4, ifdk_filter)

SEED = 20261017


def gen(spec, s0, n):
    raw = torch.empty((n, spec.Nv, spec.Nu), device="cuda")
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                      synth.default_ellipsoids(spec), s0, n, 0, spec.Nv, raw.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
    return raw


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3


def main():
    out = {}
    kinds = {"production": lambda g, Q, v: ifdk_backproject(g, Q, 0, v),
             "alg2_software": lambda g, Q, v: ifdk_backproject_alg2(g, Q, 0, v, texture=False),
             "alg2_texture": lambda g, Q, v: ifdk_backproject_alg2(g, Q, 0, v, texture=True),
             "alg4_software": lambda g, Q, v: ifdk_backproject_alg4(g, Q, 0, v, texture=False),
             "alg4_texture": lambda g, Q, v: ifdk_backproject_alg4(g, Q, 0, v, texture=True)}
    # timing: 256 views of configs 3 and 4
    for cfg in (3, 4):
        spec = synth.config(cfg)
        g = Geometry.from_spec(spec)
        raw = gen(spec, 0, 256)
        Q = torch.empty_like(raw)
        ifdk_filter(g, raw, Q)
        del raw
        vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
        for k, fn in kinds.items():
            s = timed(lambda: fn(g, Q, vol))
            ups = spec.Nx * spec.Ny * spec.Nz * 256
            out[f"config{cfg}_256views_{k}_gups"] = ups / s / 2 ** 30
            print(f"config {cfg} 256 views {k}: {s * 1e3:.1f} ms = {ups / s / 2**30:.1f} GUPS",
                  flush=True)
        del Q, vol
        torch.cuda.empty_cache()
    # accuracy: config 3 whole scan, central-plane sample vs the oracle
    spec = synth.config(3)
    g = Geometry.from_spec(spec)
    raw = gen(spec, 0, spec.Np)
    Q = torch.empty_like(raw)
    ifdk_filter(g, raw, Q)
    rng = np.random.default_rng(SEED)
    cz = spec.Nz // 2
    ijk = np.stack([rng.integers(0, spec.Nx, 1 << 13), rng.integers(0, spec.Ny, 1 << 13),
                    rng.integers(cz - 24, cz + 24, 1 << 13)], 1).astype(np.int32)
    lo, hi = 1 << 30, -1
    for s in range(spec.Np):
        a, b = g.band_rows(int(ijk[:, 2].min()), int(ijk[:, 2].max() - ijk[:, 2].min() + 1), s)
        lo, hi = min(lo, a), max(hi, b)
    og = oracle.OracleGeometry(**spec.geometry_args())
    t0 = time.time()
    Qo = oracle.filter_fft(og, raw[:, lo:hi + 1, :].cpu().numpy(), v0=lo)
    ref = oracle.backproject(og, Qo, ijk, s0=0, v0=lo)
    print(f"oracle sample: {time.time() - t0:.1f} s", flush=True)
    del raw
    idx = torch.from_numpy(ijk.astype(np.int64)).cuda()
    vol = torch.empty((spec.Nz, spec.Ny, spec.Nx), device="cuda")
    for k, fn in kinds.items():
        fn(g, Q, vol)
        got = vol[idx[:, 2], idx[:, 1], idx[:, 0]].cpu().numpy().astype(np.float64)
        d = got - ref
        rr = float(np.sqrt(np.sum(d * d) / np.sum(ref * ref)))
        mr = float(np.abs(d).max() / np.abs(ref).max())
        out[f"config3_sample_{k}_relRMSE"] = rr
        out[f"config3_sample_{k}_maxrel"] = mr
        print(f"config 3 sample {k}: relRMSE {rr:.3e}  max|d|/max|ref| {mr:.3e}", flush=True)
    with open("gpurun_out/baselines.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
