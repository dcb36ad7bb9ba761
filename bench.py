"""bench.py -- FDK (filter + back-projection) throughput on 1..8 B200s, one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of the whole hot path -- cosine weight + ramp filter of every
projection and back-projection of all of them into the volume -- over the config's
synthetic Shepp-Logan projections (BASELINE.json configs; default config 4:
2048 projections of 2048^2 -> 2048^3, which fits one GPU).  The metric is GUPS
(N_x N_y N_z N_p / (T 2^30)) for the whole step plus its end-to-end
seconds.  N > 1 runs the k-slab split (dist.kslab_reconstruct) under torchrun:
every rank filters its own views, the filter stores each row band straight into the
ranks that need it (CUDA-IPC peer memory over NVLink with device-side signals;
`--exchange nccl`: an NCCL all-to-all), each rank back-projects its slab; the step time is the max over ranks
(CUDA events + barrier).  `--impl reference` times the fp64 CPU oracle (oracle/) on a
bounded sample.

Besides the contract keys the line carries: `roofline` (BP against the measured
shared-memory gather peak, with ncu DRAM traffic), `roofline_hbm`, `roofline_issue`,
`filter_roofline`, `e2e` through the C ABI with its `host_legs`, `cpu_baseline` (oracle),
`other_configs` (configs 1-3 and config 5's per-rank slab at N = 1), `iterative` (one
config-3 SIRT iteration and the forward projector) and, at N > 1, `stage_ms` and
`variants` (projection split, R x C grid).
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

SMEM_BYTES_PER_UPDATE = 16  # 4 bilinear taps x 4 B (Alg. alg:subpixel), SURVEY 8(d)'s figure
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
    ap.add_argument("--no-oracle-full", action="store_true",
                    help="skip the full config-2 oracle run (~70 s on 16 cores) in cpu_baseline")
    ap.add_argument("--exchange", default="auto", choices=["auto", "p2p", "nccl"],
                    help="k-slab band exchange: fused filter + peer-memory scatter (auto/p2p) "
                         "or NCCL all-to-all")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip timing configs 1-3 at N = 1")
    ap.add_argument("--no-iterative", action="store_true",
                    help="skip the SIRT iteration timing on config 3")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the projection-split measurement at N > 1")
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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ncu_field(config: int, key: str):
    p = os.path.join(ROOT, "profiles", "ncu_bp_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            e = json.load(f).get(str(config))
        return e.get(key) if e else None
    return None


def walk_smem_bytes(spec):
    """Algorithmic shared-memory bytes per update and kernel of the k-walk the library picks
    for the geometry: per 64-slice chunk and view a thread issues LDS.32
    taps -- QUAD (0.5 <= dv/dk < 1): eight 4+4-slice groups x 20 taps = 640 B / 64 updates =
    10 B; QUINT (dv/dk < 0.5): six 5+5-slice groups x 16 taps + a 2+2-slice tail x 12 taps =
    432 B / 64 = 6.75 B; PAIR: 12 taps per 4 updates = 12 B."""
    import math

    r = math.hypot(spec.Nx * spec.Dx, spec.Ny * spec.Dy) / 2
    dv = [spec.D / spec.Dv * spec.Dz / z for z in (spec.d + r, spec.d - r)]
    if min(dv) >= 0.5001 and max(dv) < 0.9999:
        return 10.0, "QUAD", "bp_quad2_kernel"
    if max(dv) < 0.4999:
        return 6.75, "QUINT", "bp_quad2_kernel"
    return 12.0, "PAIR", "bp_raw_kernel"


def smem_probe():
    """Measured shared-memory gather bandwidth (bytes/s) from libifdk_probe.so, or None."""
    import ctypes

    path = os.path.join(ROOT, "paper_1909_02724_b200", "libifdk_probe.so")
    if not os.path.exists(path):
        return None, None
    lib = ctypes.CDLL(path)
    lib.ifdk_probe_smem_bandwidth.argtypes = [ctypes.POINTER(ctypes.c_double)] * 2
    lib.ifdk_probe_smem_bandwidth.restype = ctypes.c_int
    bw, ms = ctypes.c_double(), ctypes.c_double()
    if lib.ifdk_probe_smem_bandwidth(ctypes.byref(bw), ctypes.byref(ms)) != 0:
        return None, None
    return bw.value, ms.value


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
        "config": {"workload": spec.name, "config_id": args.config,
                   "Np": spec.Np, "Nu": spec.Nu, "Nv": spec.Nv,
                   "volume": [spec.Nx, spec.Ny, spec.Nz],
                   "parallelism": "host cores (fp64 oracle, OpenMP over voxels)",
                   "l2": "n/a (CPU); a bounded sample of the workload per step"},
        "cpu_baseline": {"value": value, "unit": "GUPS", "cores": cores, "kind": "oracle",
                         "sample": desc, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(out)


# ----------------------------------------------------------------------------- GPU arm
def _max_over_ranks(x, world, dev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def kslab_cross_check(g, spec, vol, k0, nk, ell, dev):
    """Max |slab - recomputation| / max |recomputation| over the first and last 64 slices of
    the slab k0..k0+nk-1 (see run_ours)."""
    import torch

    import synth
    from paper_1909_02724_b200 import ifdk_backproject, ifdk_filter
    from paper_1909_02724_b200.dist import band_union

    worst, checked = 0.0, []
    for a in sorted({k0, max(k0, k0 + nk - 64)}):
        m = min(64, k0 + nk - a)
        lo, hi = band_union(g, a, m, 0, spec.Np)
        E = torch.empty((spec.Np, hi - lo + 1, spec.Nu), device=dev)
        synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, 0,
                          spec.Np, lo, hi - lo + 1, E.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
        ifdk_filter(g, E, E, v0=lo)
        ref = torch.empty((m, spec.Ny, spec.Nx), device=dev)
        ifdk_backproject(g, E, 0, ref, k0=a, v0=lo)
        d = float((vol[a - k0:a - k0 + m] - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
        worst = max(worst, d)
        checked.append([a, m])
        del E, ref
    torch.cuda.empty_cache()
    return {"slices": checked, "max_rel_diff": worst, "tolerance": 1e-5,
            "ok": worst <= 1e-5,
            "what": "each rank's first / last 64 slices vs an exchange-free recomputation "
                    "(own row band generated on the device, filter + BP on this GPU)"}


def run_ours(args, spec, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synth
    from paper_1909_02724_b200 import (Geometry, ifdk_backproject, ifdk_filter,
                                       ifdk_reconstruct_host, last_launch_count)
    from paper_1909_02724_b200.dist import (GridPlan, SlabPlan, grid_groups, hybrid_reconstruct,
                                            kslab_reconstruct, kslab_reconstruct_host,
                                            projection_split_reconstruct)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    g = Geometry.from_spec(spec)
    plan = SlabPlan(world, spec.Nz, spec.Np)
    k0, nk = plan.slab(rank)
    stream = torch.cuda.current_stream()
    use_kslab = world > 1 or args.path == "kslab"

    # Inputs: this rank's raw views (all of them on one GPU; its 128-view blocks under the
    # k-slab split), analytic projections generated on the device.
    blocks = plan.local_views(rank) if use_kslab else [(0, spec.Np)]
    n_local = sum(n for _, n in blocks)
    raw = torch.empty((n_local, spec.Nv, spec.Nu), device=dev, dtype=torch.float32)
    ell = synth.default_ellipsoids(spec)
    off = 0
    for s0, n in blocks:
        synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell,
                          s0, n, 0, spec.Nv, raw[off:off + n].data_ptr(), stream.cuda_stream)
        off += n
    vol = torch.empty((nk, spec.Ny, spec.Nx), device=dev, dtype=torch.float32)
    batch = 256
    Q = torch.empty((min(batch, n_local), spec.Nv, spec.Nu), device=dev, dtype=torch.float32) \
        if not use_kslab else None

    bp_events = []
    filter_events = []

    def step_single(record):
        """One GPU: per 256-view batch, ifdk_filter then ifdk_backproject, with CUDA events
        around every launch.  (ifdk_reconstruct filters batch b + 1 on a side stream while
        batch b back-projects; measured the same here -- 2188 vs 2187 GUPS, the filter CTAs only
        find room as back-projection CTAs retire -- and serial launches keep the per-kernel
        timings clean.)"""
        launches = 0
        for b0 in range(0, n_local, batch):
            nb = min(batch, n_local - b0)
            q = Q[:nb]
            if record:
                f0, e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                f0.record()
            ifdk_filter(g, raw[b0:b0 + nb], q)
            launches += last_launch_count()
            if record:
                e0.record()
            ifdk_backproject(g, q, b0, vol, accumulate=b0 > 0)
            launches += last_launch_count()
            if record:
                e1.record()
                bp_events.append((e0, e1, nb))
                filter_events.append((f0, e0, nb))
        return launches

    timings = {}
    counter = [0]

    def f_fn(r, out):
        ifdk_filter(g, r, out)
        counter[0] += last_launch_count()

    def b_fn(Qb, s0, v, kk0, v0, acc):
        ifdk_backproject(g, Qb, s0, v, k0=kk0, v0=v0, accumulate=acc)
        counter[0] += last_launch_count()

    def step_multi(record):
        counter[0] = 0
        kslab_reconstruct(g, raw, vol, plan, rank, filter_fn=f_fn, bp_fn=b_fn,
                          timings=timings if record else None, force_exchange=True,
                          exchange=args.exchange)
        return counter[0]

    step = step_multi if use_kslab else step_single

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    # The BP roofline denominator, measured now (clocks warm) with the BP kernel's occupancy.
    smem_bw, _ = smem_probe()
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
    stage = {}
    for _ in range(args.steps):
        launches += step(True)
        for k, v in timings.items():
            if isinstance(v, (int, float)):
                stage[k] = stage.get(k, 0.0) + v
            else:  # labels (e.g. which exchange ran)
                stage[k] = v
    t_end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = _max_over_ranks(t_start.elapsed_time(t_end) / args.steps, world, dev)
    stage = {k: (v / args.steps if isinstance(v, (int, float)) else v) for k, v in stage.items()}

    # Dominant kernel: the back-projection; algorithmic smem bytes / its launch duration.
    if bp_events:
        dur = [a.elapsed_time(b) / 1e3 for a, b, _ in bp_events]
        n_updates = [spec.Nx * spec.Ny * nk * nb for _, _, nb in bp_events]
        bp_s = sum(dur) / len(dur)
        upd_per_launch = sum(n_updates) / len(n_updates)
        bp_share = sum(dur) / (ms / 1e3 * args.steps)
    else:  # k-slab driver: per-round BP spans (plan.world launches of 128 views each)
        bp_s = stage.get("bp_ms", float("nan")) / 1e3 / max(plan.n_rounds, 1)
        upd_per_launch = spec.Nx * spec.Ny * nk * spec.Np / max(plan.n_rounds, 1)
        bp_share = stage.get("bp_ms", float("nan")) / ms
    walk_b, walk_name, bp_kernel = walk_smem_bytes(spec)
    achieved_gbs = walk_b * upd_per_launch / bp_s / 1e9
    achieved_4tap_gbs = SMEM_BYTES_PER_UPDATE * upd_per_launch / bp_s / 1e9
    hbm_peak = float(measured_peaks().get("hbm_gbs", 6543.4))
    # BP against HBM: algorithmic bytes of one launch = its filtered views read once + the
    # slab written (first launch) or read and written (accumulating launches): 8 B per voxel
    # per launch in the steady state.
    views_per_launch = upd_per_launch / (spec.Nx * spec.Ny * nk)
    bp_hbm_bytes = 4 * views_per_launch * spec.Nu * spec.Nv + 8 * spec.Nx * spec.Ny * nk
    roofline_hbm = {"bound": "hbm", "achieved": bp_hbm_bytes / bp_s / 1e9, "peak": hbm_peak,
                    "unit": "GB/s", "frac": bp_hbm_bytes / bp_s / 1e9 / hbm_peak,
                    "kernel": f"{bp_kernel} (4 B per filtered pixel + 8 B per voxel per launch)",
                    "peak_basis": "MEASURED_PEAKS.json hbm_gbs"}
    # BP against the issue roofline: SASS instructions per update from the committed ncu
    # capture (profiles/ncu_bp_traffic.json "inst_per_update") x updates/s, against
    # 148 SMs x 4 schedulers x 32 lanes x the SM clock.
    roofline_issue = None
    ipu = ncu_field(args.config, "inst_per_update")
    if ipu:
        sm_hz = float(measured_peaks().get("sm_max_mhz", 1965.0)) * 1e6
        peak_ti = 148 * 4 * 32 * sm_hz / 1e12  # thread-instructions per second, x1e12
        ach_ti = ipu * upd_per_launch / bp_s / 1e12
        roofline_issue = {"bound": "issue", "achieved": ach_ti, "peak": peak_ti,
                          "unit": "Tinst/s (thread)", "frac": ach_ti / peak_ti,
                          "inst_per_update": ipu,
                          "kernel": bp_kernel,
                          "peak_basis": "148 SM x 4 x 32 x sm_max_mhz; inst_per_update from the "
                                        "committed ncu capture (profiles/ncu_bp_traffic.json)"}
    filt = None
    if filter_events:
        fdur = sum(a.elapsed_time(b) for a, b, _ in filter_events) / len(filter_events) / 1e3
        fpix = sum(nb for _, _, nb in filter_events) / len(filter_events) * spec.Nu * spec.Nv
        filt = {"kernel": "filter_f4k_kernel (cosine weight + ramp FFT filter)",
                "ms_per_launch": fdur * 1e3, "bound": "hbm",
                "achieved": 8 * fpix / fdur / 1e9, "peak": hbm_peak, "unit": "GB/s",
                "frac": 8 * fpix / fdur / 1e9 / hbm_peak,
                "note": "8 algorithmic B/pixel (read E, write Q); the kernel is FP32-issue "
                        "bound by the FFT's instructions (DESIGN.md section 7)"}
    derived_gbs = N_SM * SMEM_B_PER_CLK_PER_SM * 1965e6 / 1e9  # guide: 128 B/clk/SM at max clock
    if smem_bw:
        peak_gbs = smem_bw / 1e9
        peak_basis = (f"measured: conflict-free LDS.64 gather micro-benchmark (libifdk_probe, "
                      f"2 CTAs x 256 threads per SM) = {peak_gbs:.0f} GB/s; derived "
                      f"148 SM x 128 B/clk x 1965 MHz = {derived_gbs:.0f} GB/s")
    else:
        peak_gbs = derived_gbs
        peak_basis = "derived: 148 SM x 128 B/clk x 1965 MHz (probe unavailable)"
    bp_gups = upd_per_launch / bp_s / 2 ** 30
    if use_kslab and stage.get("wall_ms"):
        # delta: sum of the stage times over the wall time of the pipelined step
        stage["delta"] = (stage.get("filter_pack_ms", 0) + stage.get("bp_ms", 0)) / stage["wall_ms"]

    # At N > 1 (or the forced k-slab path) every rank cross-checks the first and last 64
    # slices of its slab against an exchange-free recomputation: the detector row band those
    # slices need, generated on the device for all views, filtered and back-projected by this
    # GPU alone.  A band routed to the wrong rank or offset would show as a gross error; the
    # filter pairs rows differently, so equality is to fp32 rounding, not bitwise.  (bench.py
    # runs the fp64 oracle only in its cpu_baseline leg; the oracle parity of this driver is
    # tests/test_gpu_dist.py.)
    slab_check = None
    if use_kslab:
        slab_check = kslab_cross_check(g, spec, vol, k0, nk, ell, dev)
        slab_check["max_rel_diff"] = _max_over_ranks(slab_check["max_rel_diff"], world, dev)

    # End to end through the public API: H2D of the raw projections from pinned host memory
    # and D2H of the volume inside the timed region, every step.
    e2e = None
    if not args.no_e2e:
        if Q is not None:
            del Q
        torch.cuda.empty_cache()
        raw_h = torch.empty(raw.shape, dtype=torch.float32, pin_memory=True)
        raw_h.copy_(raw)
        vol_h = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
        n_e2e = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 2)
        if not use_kslab:
            del raw
            torch.cuda.empty_cache()
            ifdk_reconstruct_host(g, raw_h, vol_h)  # warm-up (scratch pool, tables)
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                ifdk_reconstruct_host(g, raw_h, vol_h)
            e2e_s = (time.perf_counter() - t0) / n_e2e
            api = "ifdk_reconstruct_host (C ABI)"
        else:
            kslab_reconstruct_host(g, raw_h, vol, vol_h, plan, rank, force_exchange=True,
                                   exchange=args.exchange)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                kslab_reconstruct_host(g, raw_h, vol, vol_h, plan, rank, force_exchange=True,
                                   exchange=args.exchange)
            torch.cuda.synchronize()
            e2e_s = _max_over_ranks((time.perf_counter() - t0) / n_e2e, world, dev)
            api = "dist.kslab_reconstruct_host (per rank: H2D of its blocks, D2H of its slab)"
        h2d = _max_over_ranks(float(raw_h.numel() * 4), world, dev) * world
        d2h = _max_over_ranks(float(vol_h.numel() * 4), world, dev) * world
        e2e = {"value": gups(spec, e2e_s), "unit": "GUPS", "seconds": e2e_s,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": n_e2e, "api": api}
        # The host legs alone (pinned memory, 4 GiB each way through the same buffers), to
        # state how much of them the pipeline hides: serial = device step + H2D + D2H.
        try:
            n = min(vol.numel(), raw_h.numel(), 1 << 30)
            dv, rh, vh = vol.view(-1)[:n], raw_h.view(-1)[:n], vol_h.view(-1)[:n]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dv.copy_(rh, non_blocking=True)
            a.record()
            dv.copy_(rh, non_blocking=True)
            b.record()
            b.synchronize()
            h2d_gbs = 4 * n / (a.elapsed_time(b) / 1e3) / 1e9
            a.record()
            vh.copy_(dv, non_blocking=True)
            b.record()
            b.synchronize()
            d2h_gbs = 4 * n / (a.elapsed_time(b) / 1e3) / 1e9
            legs_s = h2d / world / 1e9 / h2d_gbs + d2h / world / 1e9 / d2h_gbs
            e2e["host_legs"] = {"h2d_gbs": h2d_gbs, "d2h_gbs": d2h_gbs,
                                "serial_seconds": ms / 1e3 + legs_s,
                                "hidden_fraction": max(0.0, 1 - (e2e_s - ms / 1e3) / legs_s)}
        except Exception as exc:  # noqa: BLE001 -- a report, never a reason to fail the bench
            e2e["host_legs"] = {"error": repr(exc)[:200]}
        del raw_h, vol_h

    # The projection-split and R x C grid variants, measured against the slab split in the
    # same run (a failure is reported in the line instead of losing it).
    variants = {}

    def measure_variants():
        nonlocal raw
        if world > 1 and not args.no_variants:
            # fused projection split: each rank back-projects its own views over the whole
            # volume and adds every 128-view partial sum straight into the owner's slab over
            # NVLink (ifdk_backproject_reduce into CUDA-IPC mappings) -- no partial volume, no
            # reduce-scatter; needs only the rank's filtered views and its own slab
            from paper_1909_02724_b200.dist import ReduceSlabs, projection_split_fused

            torch.cuda.empty_cache()
            slabs = ReduceSlabs.create(None, rank, world, g, plan.k_bounds)
            projection_split_fused(g, raw, blocks, slabs)  # warm-up
            tm = {}
            projection_split_fused(g, raw, blocks, slabs, timings=tm)
            fms = _max_over_ranks(tm["wall_ms"], world, dev)
            own = slabs.slab()
            vmax = _max_over_ranks(float(vol.abs().max()), world, dev)
            dmax = float((own - vol).abs().max()) if own.shape == vol.shape else float("nan")
            variants["projection_split_fused"] = {
                "value": gups(spec, fms / 1e3), "unit": "GUPS", "ms_per_step": fms,
                "filter_ms": _max_over_ranks(tm["filter_ms"], world, dev),
                "bp_reduce_ms": _max_over_ranks(tm["bp_reduce_ms"], world, dev),
                "max_abs_diff_vs_kslab_rel": _max_over_ranks(dmax, world, dev) / vmax,
                "what": "ifdk_backproject_reduce: red.global.add into the owners' slabs"}
            del own
            dist.barrier()
            slabs.close()
        if world > 1 and not args.no_variants and spec.Nz % world == 0:
            torch.cuda.empty_cache()
            need = 4 * (spec.Nz * spec.Ny * spec.Nx + n_local * spec.Nv * spec.Nu)
            free = torch.cuda.mem_get_info(dev)[0]
            ok = _max_over_ranks(0.0 if free > 1.05 * need else 1.0, world, dev) == 0.0
            if ok:
                ps = torch.empty((spec.Nz // world, spec.Ny, spec.Nx), device=dev)
                projection_split_reconstruct(g, raw, blocks, ps, world)  # warm-up
                tm = {}
                torch.cuda.synchronize()
                dist.barrier()
                projection_split_reconstruct(g, raw, blocks, ps, world, timings=tm)
                pms = _max_over_ranks(tm["wall_ms"], world, dev)
                same = (k0, nk) == (rank * spec.Nz // world, spec.Nz // world)
                dmax = float((ps - vol).abs().max()) if same else float("nan")
                vmax = _max_over_ranks(float(vol.abs().max()), world, dev)
                variants["projection_split"] = {
                    "value": gups(spec, pms / 1e3), "unit": "GUPS", "ms_per_step": pms,
                    "reduce_scatter_ms": _max_over_ranks(tm["reduce_scatter_ms"], world, dev),
                    "max_abs_diff_vs_kslab_rel": _max_over_ranks(dmax, world, dev) / vmax}
                del ps
            else:
                variants["projection_split"] = {"skipped": "full partial volume does not fit"}
            if world >= 4 and world % 2 == 0:
                # the paper's R x C grid with C = 2 view columns (band exchange inside a column,
                # reduce-scatter across a row); its own view blocks are generated for it
                R, C = world // 2, 2
                grid = GridPlan(R, C, spec.Nz, spec.Np)
                rows, cols = grid_groups(grid)
                gr, gc = grid.coords(rank)
                gblocks = grid.column_plan(gc).local_views(gr)
                del raw
                torch.cuda.empty_cache()
                graw = torch.empty((sum(n for _, n in gblocks), spec.Nv, spec.Nu), device=dev)
                off = 0
                for s0, n in gblocks:
                    synth.project_gpu(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta,
                                      ell, s0, n, 0, spec.Nv, graw[off:off + n].data_ptr(),
                                      torch.cuda.current_stream().cuda_stream)
                    off += n
                sk0, sn = grid.sub_slab(rank)
                gvol = torch.empty((max(sn, 1), spec.Ny, spec.Nx), device=dev)
                hybrid_reconstruct(g, graw, gvol[:sn], grid, rank, rows[gr], cols[gc])  # warm-up
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                hybrid_reconstruct(g, graw, gvol[:sn], grid, rank, rows[gr], cols[gc])
                e1.record()
                e1.synchronize()
                hms = _max_over_ranks(e0.elapsed_time(e1), world, dev)
                # cross-check against the k-slab result where the two partitions overlap
                a, b = max(sk0, k0), min(sk0 + sn, k0 + nk)
                dmax = float((gvol[a - sk0:b - sk0] - vol[a - k0:b - k0]).abs().max()) if b > a else 0.0
                vmax = _max_over_ranks(float(vol.abs().max()), world, dev)
                variants[f"grid_{R}x{C}"] = {
                    "value": gups(spec, hms / 1e3), "unit": "GUPS", "ms_per_step": hms,
                    "max_abs_diff_vs_kslab_rel": _max_over_ranks(dmax, world, dev) / vmax}
                del graw, gvol


    if world > 1 and not args.no_variants:
        try:
            measure_variants()
        except Exception as exc:  # noqa: BLE001
            variants["error"] = repr(exc)[:300]
    # The smaller configs on the same GPU (device-resident raw views, ifdk_reconstruct, median
    # of 3 after a warm-up): config 1 is latency-bound (no roofline claim), 2 and 3 full size.
    others = {}
    if world == 1 and not args.no_other_configs:
        from paper_1909_02724_b200 import ifdk_reconstruct

        for oc in (1, 2, 3):
            if oc == args.config:
                continue
            os_ = synth.config(oc)
            og_ = Geometry.from_spec(os_)
            oraw = torch.empty((os_.Np, os_.Nv, os_.Nu), device=dev)
            synth.project_gpu(os_.Nu, os_.Nv, os_.Du, os_.Dv, os_.D, os_.d, os_.theta,
                              synth.default_ellipsoids(os_), 0, os_.Np, 0, os_.Nv,
                              oraw.data_ptr(), stream.cuda_stream)
            ovol = torch.empty((os_.Nz, os_.Ny, os_.Nx), device=dev)
            ifdk_reconstruct(og_, oraw, ovol)
            ts = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ifdk_reconstruct(og_, oraw, ovol)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            t_ms = sorted(ts)[1]
            others[os_.name] = {"fdk_ms": t_ms, "gups": gups(os_, t_ms / 1e3),
                                "kernel_launches": last_launch_count()}
            del oraw, ovol
        torch.cuda.empty_cache()
        # Config 5 (4096 views of 2048^2 -> 4096^3, 256 GiB) only exists k-slab-partitioned over
        # 8 GPUs; one GPU runs one rank's share: slab 0 (512 slices) from its row band, the
        # first 256 views (filter + BP through the C ABI).
        if args.config != 5:
            from paper_1909_02724_b200 import ifdk_backproject, ifdk_filter

            c5 = synth.config(5)
            g5 = Geometry.from_spec(c5)
            k0, nk, n5 = 0, c5.Nz // 8, 256
            lo = min(g5.band_rows(k0, nk, s5)[0] for s5 in range(n5))
            hi = max(g5.band_rows(k0, nk, s5)[1] for s5 in range(n5))
            e5 = torch.empty((n5, hi - lo + 1, c5.Nu), device=dev)
            synth.project_gpu(c5.Nu, c5.Nv, c5.Du, c5.Dv, c5.D, c5.d, c5.theta,
                              synth.default_ellipsoids(c5), 0, n5, lo, hi - lo + 1,
                              e5.data_ptr(), stream.cuda_stream)
            v5 = torch.empty((nk, c5.Ny, c5.Nx), device=dev)
            ts = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                q5 = e5.clone()
                a.record()
                ifdk_filter(g5, q5, q5, v0=lo)
                ifdk_backproject(g5, q5, 0, v5, k0=k0, v0=lo)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
                del q5
            t_ms = sorted(ts)[1]
            others[f"{c5.name} (k-slab 0 of 8, 256 views)"] = {
                "fdk_ms": t_ms, "gups": c5.Nx * c5.Ny * nk * n5 / (t_ms / 1e3) / 2 ** 30,
                "band_rows": hi - lo + 1, "kernel_launches": 2}
            del e5, v5
            torch.cuda.empty_cache()

    # Iterative reconstruction: one SIRT iteration on config 3 (1024 views
    # of 1024^2 -> 1024^3) = forward projection + back-projection + element-wise steps, the
    # normalisers precomputed; the forward projector timed alone as well (GUPS = voxel-view
    # splats per second).  Measured projections = the analytic phantom's.
    iterative = None
    if world == 1 and not args.no_iterative:
        from paper_1909_02724_b200 import SART, ifdk_fill, ifdk_forward_project

        is_ = synth.config(3)
        ig = Geometry.from_spec(is_)
        ib = torch.empty((is_.Np, is_.Nv, is_.Nu), device=dev)
        synth.project_gpu(is_.Nu, is_.Nv, is_.Du, is_.Dv, is_.D, is_.d, is_.theta,
                          synth.default_ellipsoids(is_), 0, is_.Np, 0, is_.Nv,
                          ib.data_ptr(), stream.cuda_stream)
        st = SART(ig, ib)
        ix = torch.empty((is_.Nz, is_.Ny, is_.Nx), device=dev)
        ifdk_fill(ix, 0.0)
        st.iterate(ix, 1)  # warm-up
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.iterate(ix, 2)
        b.record()
        b.synchronize()
        it_ms = a.elapsed_time(b) / 2
        a.record()
        ifdk_forward_project(ig, ix, 0, ib)
        b.record()
        b.synchronize()
        fp_ms = a.elapsed_time(b)
        it_launches = last_launch_count()
        iterative = {"workload": f"SIRT {is_.name}", "seconds_per_iteration": it_ms / 1e3,
                     "fp_ms": fp_ms, "fp_gups": gups(is_, fp_ms / 1e3),
                     "fp_kernel_launches": it_launches,
                     "note": "one iteration = forward projection + ratio + back-projection + "
                             "update over all 1024 views; normalisers R = M1, C = M^T 1 "
                             "precomputed (DESIGN.md section 13)"}
        del ib, ix, st
        torch.cuda.empty_cache()

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle

        oracle.build()
        v, s, desc = oracle_sample(spec, 32, 1 << 25)  # ~10-20 s on the box's 16 cores
        cpu = {"value": v, "unit": "GUPS", "cores": oracle.num_threads(), "kind": "oracle",
               "sample": desc, "seconds": s, "cpu_model": cpu_model()}
        cpu["updates_per_s_per_core"] = v * 2 ** 30 / cpu["cores"]
        # configs 1 and 2 in full, not extrapolated: oracle filter (direct sum for
        # config 1, FFT form for config 2) + back-projection of every voxel over every view
        for cid, fft in ((1, False), (2, True)):
            if args.no_oracle_full and cid == 2:
                continue
            c = synth.config(cid)
            Ec = synth.project(c.Nu, c.Nv, c.Du, c.Dv, c.D, c.d, c.theta,
                               synth.default_ellipsoids(c), 0, c.Np)
            t1 = time.perf_counter()
            oracle.reconstruct(oracle.OracleGeometry(**c.geometry_args()), Ec, fft=fft)
            dt = time.perf_counter() - t1
            cpu[f"config{cid}_full"] = {"workload": c.name, "seconds": dt,
                                        "gups": gups(c, dt),
                                        "updates_per_s_per_core": c.updates / dt / cpu["cores"],
                                        "measured": "in full (every voxel, every view)"}
            del Ec
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
                   "parallelism": (f"k-slab x{world} (pipelined 128-view rounds, band exchange: "
                                  f"{stage.get('exchange', 'none')})") if use_kslab
                                 else "single GPU",
                   "l2": f"projections ({4 * spec.Np * spec.Nu * spec.Nv / 2**30:.0f} GiB) and "
                         f"volume ({4 * spec.Nx * spec.Ny * spec.Nz / 2**30:.0f} GiB) far larger "
                         "than the 126 MB L2; no flush"},
        "bp_gups": bp_gups,
        "bp_share_of_step": bp_share,
        "roofline": {"bound": "smem", "achieved": achieved_gbs, "peak": peak_gbs,
                     "unit": "GB/s", "frac": achieved_gbs / peak_gbs,
                     "frac_vs_derived_peak": achieved_gbs / derived_gbs,
                     # per launch, scaled by updates from the captured 256-view full-depth
                     # launch (k-slab rounds at N > 1 are smaller launches)
                     "traffic": (ncu_traffic(args.config) * upd_per_launch
                                 / (256.0 * spec.Nx * spec.Ny * spec.Nz)
                                 if ncu_traffic(args.config) else None),
                     "bytes_per_update": walk_b,
                     "kernel": f"{bp_kernel} ({walk_name} walk: {walk_b} algorithmic B/update "
                               "of shared-memory taps; TMEM accumulators, two views per step)",
                     "smem_bytes_per_update_ncu": ncu_field(args.config, "smem_bytes_per_update"),
                     "four_tap": {"bytes_per_update": SMEM_BYTES_PER_UPDATE,
                                  "achieved": achieved_4tap_gbs,
                                  "frac": achieved_4tap_gbs / peak_gbs,
                                  "note": "SURVEY 8(d)'s 4-tap figure; the walk reuses detector "
                                          "rows across slices, so it moves fewer bytes and this "
                                          "fraction can exceed 1"},
                     "peak_basis": peak_basis},
        "roofline_hbm": roofline_hbm,
        "roofline_issue": roofline_issue,
        "filter_roofline": filt,
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches,
        "cpu_baseline": cpu,
    }
    if stage:
        out["stage_ms"] = stage
    if slab_check:
        out["slab_cross_check"] = slab_check
    if variants:
        out["variants"] = variants
    if others:
        out["other_configs"] = others
    if iterative:
        out["iterative"] = iterative
    emit(out)


_JSON_OUT = None


def emit(out):
    """The one JSON line, on the process's original stdout."""
    f = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    f.write(json.dumps(out) + "\n")
    f.flush()


def route_stdout_to_stderr():
    """Keep stdout for the JSON line alone: everything else written to fd 1 -- NCCL's version
    banner at process-group init, library prints -- goes to stderr."""
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def main():
    route_stdout_to_stderr()
    args = parse()
    import synth

    spec = synth.config(args.config)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, spec, rank, world)
        return
    # Under torchrun the process group exists even at N = 1 when the k-slab driver is forced,
    # so that its NCCL exchange runs on the pipeline's streams.
    use_pg = world > 1 or (args.path == "kslab" and "MASTER_ADDR" in os.environ)
    if use_pg:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, spec, rank, world, local_rank)
    finally:
        if use_pg:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
