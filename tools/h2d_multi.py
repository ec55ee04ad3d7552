"""Concurrent pinned H2D bandwidth on every visible GPU (one process per GPU under
torchrun): the e2e input path of an N-GPU step shares the host's memory / PCIe fabric.
    torchrun --nproc-per-node N tools/h2d_multi.py"""
import os

import torch
import torch.distributed as dist

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    dbuf.copy_(h, non_blocking=True)
torch.cuda.synchronize()
res = []
for _ in range(5):
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        dbuf.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    res.append(4 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
out = [None] * dist.get_world_size()
dist.all_gather_object(out, max(res))
if dist.get_rank() == 0:
    print("concurrent H2D GB/s per GPU:", [round(v, 1) for v in out], "sum", round(sum(out), 1))
