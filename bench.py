"""bench.py -- FDK (filter + back-projection) throughput on 1..8 B200s, one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of the whole hot path -- cosine weight + ramp filter of every
projection and back-projection of all of them into the volume -- over the config's
synthetic Shepp-Logan projections (BASELINE.json configs; default config 4:
2048 projections of 2048^2 -> 2048^3, which fits one GPU).  The metric is GUPS
(N_x N_y N_z N_p / (T 2^30)) for the whole step plus its end-to-end
seconds.  N > 1 runs the k-slab split (dist.kslab_reconstruct) under torchrun:
every rank filters its own views, an NCCL all-to-all moves row bands, each rank
back-projects its slab; the step time is the max over ranks (CUDA events + barrier).
`--impl reference` times the fp64 CPU oracle (oracle/) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SMEM_BYTES_PER_UPDATE = 16  # 4 bilinear taps x 4 B (Alg. alg:subpixel), DESIGN.md "Roofline"
SMEM_B_PER_CLK_PER_SM = 128
N_SM = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--path", default="auto", choices=["auto", "kslab"],
                    help="kslab forces the multi-GPU k-slab driver even at N=1")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# ----------------------------------------------------------------------------- helpers
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def ncu_traffic(config: int):
    """DRAM bytes (read + write) per bench BP launch from the committed ncu --set full capture
    (profiles/ncu_bp_traffic.json: a 256-view x 256-slice launch scaled by updates), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_bp_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        e = d.get(str(config))
        return e["bytes_per_launch"] if e else None
    return None


def gups(spec, seconds):
    return spec.updates / seconds / 2 ** 30


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample(spec, n_views: int, n_vox: int, seed: int = 20261017):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload: the FFT form
    of Alg. alg:filter on n_views whole views and Alg. alg:bp of n_vox random voxels over
    those views.  Returns (extrapolated GUPS for the whole config, seconds, description)."""
    import numpy as np

    import oracle
    import synth

    og = oracle.OracleGeometry(**spec.geometry_args())
    ell = synth.default_ellipsoids(spec)
    s0 = spec.Np // 3
    E = synth.project(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, s0,
                      n_views)
    rng = np.random.default_rng(seed)
    ijk = np.stack([rng.integers(0, n, n_vox) for n in (spec.Nx, spec.Ny, spec.Nz)], 1)
    t0 = time.perf_counter()
    Q = oracle.filter_fft(og, E)
    t1 = time.perf_counter()
    oracle.backproject(og, Q, ijk, s0=s0)
    t2 = time.perf_counter()
    n_vox_all = spec.Nx * spec.Ny * spec.Nz
    t_total = (t1 - t0) * spec.Np / n_views + (t2 - t1) * (n_vox_all / n_vox) * (spec.Np / n_views)
    desc = (f"oracle filter_fft of {n_views} whole views + oracle backproject of {n_vox} random "
            f"voxels x {n_views} views ({n_vox * n_views} updates); extrapolated to the full "
            f"config (filter x Np/{n_views}, BP x voxels x views)")
    return spec.updates / t_total / 2 ** 30, t2 - t0, desc


def run_reference(args, spec, rank, world):
    if rank != 0:
        return
    import oracle

    oracle.build()
    n_views, n_vox = 8, 1 << 23  # ~3-5 s of 16-core oracle work per step
    for _ in range(args.warmup):
        oracle_sample(spec, n_views, n_vox)
    vals, secs = [], []
    for _ in range(args.steps):
        v, s, desc = oracle_sample(spec, n_views, n_vox)
        vals.append(v)
        secs.append(s)
    value = sorted(vals)[len(vals) // 2]
    cores = oracle.num_threads()
    out = {
        "impl": "reference",
        "metric": "fdk_gups",
        "value": value,
        "unit": "GUPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * sorted(secs)[len(secs) // 2],
        "full_workload_ms_extrapolated": 1e3 * spec.updates / value / 2 ** 30,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (analytic Shepp-Logan projections, seeded)",
        "config": {"workload": spec.name, "config_id": args.config},
        "cpu_baseline": {"value": value, "unit": "GUPS", "cores": cores, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args, spec, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synth
    from paper_1909_02724_b200 import (Geometry, ifdk_backproject, ifdk_filter,
                                       ifdk_reconstruct_host, last_launch_count)
    from paper_1909_02724_b200.dist import SlabPlan, kslab_reconstruct

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    g = Geometry.from_spec(spec)
    plan = SlabPlan(world, spec.Nz, spec.Np)
    vs0, nv = plan.views(rank)
    k0, nk = plan.slab(rank)
    stream = torch.cuda.current_stream()

    # Inputs: this rank's raw views, analytic projections generated on the device.
    raw = torch.empty((nv, spec.Nv, spec.Nu), device=dev, dtype=torch.float32)
    ell = synth.default_ellipsoids(spec)
    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, vs0,
                      nv, 0, spec.Nv, raw.data_ptr(), stream.cuda_stream)
    vol = torch.empty((nk, spec.Ny, spec.Nx), device=dev, dtype=torch.float32)
    batch = 256
    Q = torch.empty((min(batch, nv), spec.Nv, spec.Nu), device=dev, dtype=torch.float32) \
        if (world == 1 and args.path == "auto") else None

    bp_events = []

    def step_single(record):
        """World 1: per 256-view batch, ifdk_filter then ifdk_backproject (what
        ifdk_reconstruct does), with CUDA events around every BP launch."""
        launches = 0
        for b0 in range(0, nv, batch):
            nb = min(batch, nv - b0)
            q = Q[:nb]
            ifdk_filter(g, raw[b0:b0 + nb], q)
            launches += last_launch_count()
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            ifdk_backproject(g, q, b0, vol, accumulate=b0 > 0)
            launches += last_launch_count()
            if record:
                e1.record()
                bp_events.append((e0, e1, nb))
        return launches

    timings = {}

    def step_multi(record):
        kslab_reconstruct(g, raw, vol, plan, rank, timings=timings if record else None)
        return 2 + world  # filter + one BP per source rank (+ NCCL)

    step = step_single if (world == 1 and args.path == "auto") else step_multi

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_start.record()
    launches = 0
    for _ in range(args.steps):
        launches += step(True)
    t_end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # Dominant kernel: the back-projection; algorithmic smem bytes / its launch duration.
    if bp_events:
        dur = [a.elapsed_time(b) / 1e3 for a, b, _ in bp_events]
        n_updates = [spec.Nx * spec.Ny * nk * nb for _, _, nb in bp_events]
        bp_s = sum(dur) / len(dur)
        upd_per_launch = sum(n_updates) / len(n_updates)
        bp_share = sum(dur) / (ms / 1e3 * args.steps)
    else:
        bp_s = timings.get("bp_ms", float("nan")) / 1e3
        upd_per_launch = spec.Nx * spec.Ny * nk * spec.Np
        bp_share = bp_s / (ms / 1e3)
    achieved_gbs = SMEM_BYTES_PER_UPDATE * upd_per_launch / bp_s / 1e9
    peak_gbs = N_SM * SMEM_B_PER_CLK_PER_SM * 1965e6 / 1e9  # at the max SM clock
    bp_gups = upd_per_launch / bp_s / 2 ** 30

    # End to end through the public host API: H2D of the raw projections from pinned host
    # memory and D2H of the volume inside the timed region, every step.
    e2e = None
    if not args.no_e2e and world == 1:
        if Q is not None:
            del Q
        torch.cuda.empty_cache()
        raw_h = torch.empty(raw.shape, dtype=torch.float32, pin_memory=True)
        raw_h.copy_(raw)
        del raw
        torch.cuda.empty_cache()
        vol_h = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
        n_e2e = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 2)
        ifdk_reconstruct_host(g, raw_h, vol_h)  # warm-up (allocator, tables)
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            ifdk_reconstruct_host(g, raw_h, vol_h)
        e2e_s = (time.perf_counter() - t0) / n_e2e
        e2e = {"value": gups(spec, e2e_s), "unit": "GUPS", "seconds": e2e_s,
               "h2d_bytes_per_step": raw_h.numel() * 4, "d2h_bytes_per_step": vol_h.numel() * 4,
               "steps": n_e2e}
    elif world > 1:
        e2e = {"value": None, "unit": "GUPS", "note": "host API e2e measured at N=1 only",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle

        oracle.build()
        v, s, desc = oracle_sample(spec, 32, 1 << 25)  # ~10-20 s on the box's 16 cores
        cpu = {"value": v, "unit": "GUPS", "cores": oracle.num_threads(), "kind": "oracle",
               "sample": desc, "seconds": s}
    value = gups(spec, ms / 1e3)
    out = {
        "metric": "fdk_gups",
        "value": value,
        "unit": "GUPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "fdk_seconds": ms / 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (analytic Shepp-Logan projections generated on the GPU, seeded)",
        "config": {"workload": spec.name, "config_id": args.config,
                   "Np": spec.Np, "Nu": spec.Nu, "Nv": spec.Nv,
                   "volume": [spec.Nx, spec.Ny, spec.Nz],
                   "parallelism": f"k-slab x{world}" if (world > 1 or args.path == "kslab")
                   else "single GPU",
                   "l2": f"projections ({4 * spec.Np * spec.Nu * spec.Nv / 2**30:.0f} GiB) and "
                         f"volume ({4 * spec.Nx * spec.Ny * spec.Nz / 2**30:.0f} GiB) far larger "
                         "than the 126 MB L2; no flush"},
        "bp_gups": bp_gups,
        "bp_share_of_step": bp_share,
        "roofline": {"bound": "smem", "achieved": achieved_gbs, "peak": peak_gbs,
                     "unit": "GB/s", "frac": achieved_gbs / peak_gbs,
                     "traffic": ncu_traffic(args.config),
                     "kernel": "bp_kernel (16 algorithmic B/update of bilinear taps)",
                     "peak_basis": "148 SM x 128 B/clk x 1965 MHz (no measured smem peak in "
                                   "MEASURED_PEAKS.json)"},
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches,
        "cpu_baseline": cpu,
    }
    if timings:
        out["stage_ms"] = timings
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    import synth

    spec = synth.config(args.config)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, spec, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, spec, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
