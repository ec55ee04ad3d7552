"""Diagnostic: eager step time after graph capture / graph e2e (not collected)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops
from paper_2407_04656_b200.graphs import GraphedStep
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias, stage_breakdown
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
dev = torch.device("cuda", 0)
E, k, d, dff, Tn = 16, 2, 1024, 4096, 65536
layer = MoELayer(d, dff, E, k, router_bias=zipf_router_bias(E, 1.2), device=dev, router_std=0.04)
x = torch.randn(Tn, d, device=dev).bfloat16()
dout = (torch.randn(Tn, d, device=dev) * 1e-2).bfloat16()
hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
layer.set_plan(replica_matrix(plan_for_loads(hist.tolist(), 1, 80, 2)))
def eager():
    layer.zero_grad(set_to_none=True)
    layer(x).backward(dout)
def tm(fn, n=10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
for _ in range(3): eager()
print("eager before graph %.2f ms" % tm(eager), flush=True)
g = GraphedStep(layer, Tn, nbuf=2)
for b in range(2):
    g.x[b].copy_(x); g.dout[b].copy_(dout)
print("graph replay %.2f ms" % tm(lambda: g.replay(0)), flush=True)
print("eager after graph %.2f ms" % tm(eager), flush=True)
layer.stage_events = []
tm(eager, 3)
print({k2: round(v / 3, 3) for k2, v in stage_breakdown(layer.stage_events).items()})
layer.stage_events = None
print("mem reserved GB %.1f allocated GB %.1f" % (torch.cuda.memory_reserved() / 1e9, torch.cuda.memory_allocated() / 1e9))
for p in layer.parameters():
    print(tuple(p.shape), None if p.grad is None else p.grad.data_ptr() % 1000)
