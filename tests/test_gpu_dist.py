"""The k-slab driver on the GPU box.

* Under torchrun with NCCL (world size = visible GPUs, 1 on the development boxes): both
  exchanges -- the fused filter + band scatter into CUDA-IPC peer memory with device-side
  signals, and the NCCL all-to-all -- and the end-to-end host form are bitwise equal to
  ifdk_reconstruct and match the oracle; the projection split (NCCL reduce-scatter) equals it
  within fp32 order.
* Virtual ranks (P = 2, 4, 8 in one process on one GPU): the production fused exchange
  layout, the scatter kernel's completion flags and the wait / signal kernels.
* Two processes on ONE GPU (gloo for the host plumbing): the fused exchange across real
  process boundaries (IPC-mapped buffers, signals between time-sliced contexts), and the
  fused projection split's adds into a peer's IPC-mapped slab.
* Virtual ranks for the fused reduce: the projection split at P = 1-8 and
  R x C grids, back-projection adding straight into the owners' slabs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_kslab_under_torchrun_both_exchanges():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = min(torch.cuda.device_count(), 8)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", "29611", os.path.join(ROOT, "tools", "kslab_check.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-3000:]
    assert out.count("bitwise=OK") == 3 * n, out[-3000:]  # auto, nccl, end-to-end host
    assert out.count("ORACLE-OK") == 2 * n, out[-3000:]
    assert out.count("PSPLIT") == n and "MISMATCH" not in out, out[-3000:]
    assert out.count("PSFUSED") == n, out[-3000:]
    # on B200 the default exchange is the fused filter + peer-memory scatter
    assert out.count("exchange=auto used=p2p-fused") == n, out[-3000:]


def test_virtual_ranks_fused_exchange():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "virtual_ranks_check.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-3000:]
    assert out.count("bitwise=OK") == 5 and "MISMATCH" not in out, out[-3000:]


def test_two_processes_one_gpu_fused_exchange():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, KSLAB_SAME_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1",
                        "--master-port", "29613", os.path.join(ROOT, "tools", "kslab_check.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-3000:]
    assert out.count("exchange=p2p used=p2p-fused bitwise=OK") == 2, out[-3000:]
    assert out.count("ORACLE-OK") == 2 and out.count("KSLAB-HOST") == 2, out[-3000:]
    assert out.count("PSFUSED") == 2, out[-3000:]
    assert "MISMATCH" not in out, out[-3000:]


def test_virtual_ranks_fused_reduce_and_grid():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "grid_check.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-3000:]
    assert out.count("OK") >= 9 and "MISMATCH" not in out, out[-3000:]
    assert out.count("FUSED projection split") == 4 and out.count("FUSED R x C grid") == 5
