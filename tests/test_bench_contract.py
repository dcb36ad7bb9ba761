"""bench.py keeps its JSON-line contract: the reference arm on CPU (-m "not gpu"), and the GPU
arm at N=1 on a small config, through both the single-GPU path and the k-slab (multi-GPU)
path under torchrun at world size 1 (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "gpu_launches", "cpu_baseline"}


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["impl"] == "reference"
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["metric"] == "fdk_gups" and d["unit"] == "GUPS" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"] == "64x64^2->64^3"


@pytest.mark.gpu
def test_gpu_arm_json_line_single_and_kslab():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    common = ["--config", "1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
              "--no-other-configs", "--no-iterative"]
    r = subprocess.run([sys.executable, "bench.py", *common], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert {"roofline", "clocks", "roofline_hbm", "filter_roofline"} <= set(d)
    assert d["gpu_launches"] > 0 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"]
    # the multi-GPU code path of bench.py (k-slab pipeline, exchange through the process
    # group) at world size 1 under torchrun
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=1", "--master-addr", "127.0.0.1", "--master-port",
                        "29547", "bench.py", "--gpus", "1", "--path", "kslab", *common],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert BASE_KEYS <= set(d) and d["value"] > 0
    assert "k-slab" in d["config"]["parallelism"]
    # the k-slab result cross-checked against an exchange-free recomputation, delta reported
    assert d["slab_cross_check"]["ok"], d["slab_cross_check"]
    assert d["stage_ms"]["delta"] > 0
