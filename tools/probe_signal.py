"""Probe of the device-side signals on one GPU (debug aid for the fused exchange): a wait
kernel enqueued on one stream before the signal it needs is enqueued on another.
Each case prints OK or STUCK (the wait kernel traps after 20 s)."""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_02724_b200.ifdk import as_tensor, ifdk_signal, ifdk_wait, peer_alloc  # noqa: E402


def new_stream():
    from cuda.bindings import runtime as cudart

    err, s = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
    return torch.cuda.ExternalStream(int(s))


def run(name, n_streams, wait_idx, sig_idx, use_pool=False):
    ptr, _ = peer_alloc(4096)
    as_tensor(ptr, (1024,), "uint32").zero_()
    torch.cuda.synchronize()
    ss = [torch.cuda.Stream() if use_pool else new_stream() for _ in range(n_streams)]
    with torch.cuda.stream(ss[wait_idx]):
        ifdk_wait(ptr, 1, 1, 20000)
    ev = torch.cuda.Event()
    ev.record(ss[wait_idx])
    time.sleep(0.5)
    with torch.cuda.stream(ss[sig_idx]):
        ifdk_signal([ptr])
    t0 = time.time()
    while not ev.query():
        if time.time() - t0 > 15:
            print(f"{name}: STUCK", flush=True)
            os._exit(3)
        time.sleep(0.01)
    print(f"{name}: OK {time.time() - t0:.3f} s", flush=True)


def run_scatter():
    """wait on stream 0 for the completion flag of ifdk_filter_scatter on stream 1"""
    import synth
    from paper_1909_02724_b200 import Geometry
    from paper_1909_02724_b200.ifdk import ifdk_filter_scatter

    spec = synth.ConfigSpec("p", 64, 128, 128, 64, 64, 64)
    g = Geometry.from_spec(spec)
    raw = torch.rand((64, 128, 128), device="cuda")
    out = torch.empty((64, 40, 128), device="cuda")
    ptr, _ = peer_alloc(4096)
    as_tensor(ptr, (1024,), "uint32").zero_()
    torch.cuda.synchronize()
    a, b = new_stream(), new_stream()
    with torch.cuda.stream(a):
        ifdk_wait(ptr, 2, 1, 20000)
    ev = torch.cuda.Event()
    ev.record(a)
    time.sleep(0.5)
    with torch.cuda.stream(b):
        ifdk_filter_scatter(g, raw, [(out.data_ptr(), 30, 69)], flags=[ptr, ptr + 4],
                            ticket=ptr + 512)
    t0 = time.time()
    while not ev.query():
        if time.time() - t0 > 15:
            w = as_tensor(ptr, (256,), "uint32")
            print("scatter: STUCK", flush=True)
            os._exit(3)
        time.sleep(0.01)
    torch.cuda.synchronize()
    print(f"scatter: OK {time.time() - t0:.3f} s words={as_tensor(ptr, (256,), 'uint32').cpu().tolist()[0:2]}",
          flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    case = sys.argv[1]
    if case == "2":
        run("2 streams", 2, 0, 1)
    elif case == "24":
        run("24 streams, signal on the last", 24, 0, 23)
    elif case == "40":
        run("40 streams, signal on the 33rd", 40, 0, 32)
    elif case == "scatter":
        run_scatter()
    elif case == "pool":
        run("torch pool streams", 2, 0, 1, use_pool=True)
