"""Diagnostic: where does the D2H-scalar penalty go with the CTA-pair GEMM (not collected)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias, stage_breakdown
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix

dev = torch.device("cuda", 0)
E, k, d, dff, Tn = 16, 2, 1024, 4096, 65536
layer = MoELayer(d, dff, E, k, router_bias=zipf_router_bias(E, 1.2), device=dev)
x = torch.randn(Tn, d, device=dev).bfloat16()
dout = (torch.randn(Tn, d, device=dev) * 1e-2).bfloat16()
hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
layer.set_plan(replica_matrix(plan_for_loads(hist.tolist(), 1, 48, 2)))
res = torch.empty(1).pin_memory()

def step(mode):
    layer.zero_grad(set_to_none=True)
    out = layer(x)
    out.backward(dout)
    if mode == 1:
        s = out.float().sum().view(1)
    elif mode == 2:
        s = out.float().sum().view(1)
        res.copy_(s, non_blocking=True)
    elif mode == 3:
        s = out[:1, :1].float().view(1)
        res.copy_(s, non_blocking=True)

for mode in (0, 1, 2, 3):
    for _ in range(3):
        step(mode)
    torch.cuda.synchronize()
    layer.stage_events = []
    t0 = time.perf_counter()
    for _ in range(5):
        step(mode)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    st = stage_breakdown(layer.stage_events)
    layer.stage_events = None
    print(f"mode {mode}: {dt*1e3:.2f} ms/step", {kk: round(v / 5, 3) for kk, v in st.items()}, flush=True)
