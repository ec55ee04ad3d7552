"""Diagnostic: host-side stall inside plan_device after a D2H copy (not collected)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops, dispatch as D, _lib
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix

dev = torch.device("cuda", 0)
E, k, d, dff, Tn = 16, 2, 1024, 4096, 65536
layer = MoELayer(d, dff, E, k, router_bias=zipf_router_bias(E, 1.2), device=dev)
x = torch.randn(Tn, d, device=dev).bfloat16()
dout = (torch.randn(Tn, d, device=dev) * 1e-2).bfloat16()
hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
layer.set_plan(replica_matrix(plan_for_loads(hist.tolist(), 1, 48, 2)))
res = torch.empty(1).pin_memory()
T = {}
orig_call = _lib.call
def timed_call(name, *a):
    t0 = time.perf_counter(); orig_call(name, *a); T[name] = T.get(name, 0) + time.perf_counter() - t0
_lib.call = timed_call
orig_empty = torch.empty
def step():
    layer.zero_grad(set_to_none=True)
    out = layer(x)
    out.backward(dout)
    res.copy_(out.float().sum().view(1), non_blocking=True)
for _ in range(3):
    step()
torch.cuda.synchronize()
T.clear()
t0 = time.perf_counter()
for _ in range(5):
    step()
torch.cuda.synchronize()
print("total", (time.perf_counter() - t0) / 5 * 1e3, "ms/step")
for kk, v in sorted(T.items(), key=lambda z: -z[1]):
    print(f"  {kk:28s} {v / 5 * 1e3:8.3f} ms/step host")
