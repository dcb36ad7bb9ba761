"""Probe torch symmetric memory on this box (dev aid): rendezvous, peer pointer, barrier."""
import os
import traceback

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
pg = dist.group.WORLD
print("backend", symm_mem.get_backend(torch.device("cuda", 0)) if hasattr(symm_mem, "get_backend") else "?")
for step in ("enable", "empty", "rendezvous", "barrier"):
    try:
        if step == "enable":
            symm_mem.enable_symm_mem_for_group(pg.group_name)
        elif step == "empty":
            buf = symm_mem.empty(1 << 20, dtype=torch.float32, device="cuda")
        elif step == "rendezvous":
            hdl = symm_mem.rendezvous(buf, pg)
            print("ptrs", hdl.buffer_ptrs, "rank", hdl.rank, "world", hdl.world_size)
        else:
            hdl.barrier(channel=0)
            torch.cuda.synchronize()
        print("OK", step, flush=True)
    except Exception:
        print("FAIL", step)
        traceback.print_exc()
        break
dist.destroy_process_group()
