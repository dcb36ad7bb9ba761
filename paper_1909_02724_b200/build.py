"""Build libifdk.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libifdk.so")
PROBE_LIB = os.path.join(HERE, "libifdk_probe.so")  # shared-memory roofline micro-benchmark
SOURCES = ["geometry.cpp", "filter.cu", "backproject.cu", "forward.cu", "baseline.cu", "peer.cu",
           "api.cu"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "ifdk.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build_probe(force: bool = False) -> str:
    src = os.path.join(CSRC, "probe.cu")
    if force or not os.path.exists(PROBE_LIB) or os.path.getmtime(src) > os.path.getmtime(PROBE_LIB):
        cmd = ["nvcc", *NVCC_FLAGS, "-shared", src, "-o", PROBE_LIB + ".tmp", "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libifdk_probe.so")
        os.replace(PROBE_LIB + ".tmp", PROBE_LIB)
    return PROBE_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    build_probe(force)
    if not force and not _stale():
        return LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    cmd = ["nvcc", *NVCC_FLAGS, "-shared", *srcs, "-o", LIB + ".tmp", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libifdk.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
