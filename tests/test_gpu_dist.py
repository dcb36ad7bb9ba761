"""The k-slab driver under torchrun with NCCL on the GPU box (world size = visible GPUs, 1 on
the development boxes): both exchanges -- the fused filter + NVLink band scatter over
symmetric memory and the NCCL all-to-all -- and the end-to-end host form are bitwise equal to
ifdk_reconstruct; the projection split (NCCL reduce-scatter) equals it within fp32 order."""
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
    assert out.count("PSPLIT") == n and "MISMATCH" not in out, out[-3000:]
    # on B200 the default exchange is the fused filter + symmetric-memory scatter
    assert out.count("exchange=auto used=p2p-fused") == n, out[-3000:]
