"""Pinned H2D bandwidth while the GPU runs a GEMM loop (the e2e input path competes
with the step):   python tools/h2d_load.py"""
import torch

n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(n, dtype=torch.uint8, device="cuda")
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
cs = torch.cuda.Stream()
for load in (False, True):
    for _ in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if load:
            for _ in range(40):
                torch.mm(a, b)
        with torch.cuda.stream(cs):
            e0.record(cs)
            dbuf.copy_(h, non_blocking=True)
            e1.record(cs)
        torch.cuda.synchronize()
    print(f"H2D {'under GEMM load' if load else 'idle'}: {n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
