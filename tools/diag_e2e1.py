"""Diagnostic: e2e step-time variants on one GPU (not collected by pytest)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops
from paper_2407_04656_b200.hostio import HostPrefetcher
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix

dev = torch.device("cuda", 0)
E, k, d, dff, Tn = 16, 2, 1024, 4096, 65536
layer = MoELayer(d, dff, E, k, router_bias=zipf_router_bias(E, 1.2), device=dev)
x = torch.randn(Tn, d, device=dev).bfloat16()
dout = (torch.randn(Tn, d, device=dev) * 1e-2).bfloat16()
hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
layer.set_plan(replica_matrix(plan_for_loads(hist.tolist(), 1, 48, 2)))
x_h, d_h = x.cpu().pin_memory(), dout.cpu().pin_memory()
res = torch.empty(1).pin_memory()

def step(xx, dd):
    layer.zero_grad(set_to_none=True)
    out = layer(xx)
    out.backward(dd)
    return out

def run(name, fn, K=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter() - t0) / K * 1e3:8.2f} ms/step", flush=True)

run("resident", lambda: step(x, dout))
run("resident + d2h scalar", lambda: res.copy_(step(x, dout).float().sum().view(1), non_blocking=True))
run("h2d non_blocking", lambda: step(x_h.to(dev, non_blocking=True), d_h.to(dev, non_blocking=True)))
def with_d2h():
    out = step(x_h.to(dev, non_blocking=True), d_h.to(dev, non_blocking=True))
    res.copy_(out.float().sum().view(1), non_blocking=True)
run("h2d + d2h scalar", with_d2h)
pf = HostPrefetcher([x_h, d_h], dev)
pf.prefetch()
def pref():
    xx, dd = pf.get()
    pf.prefetch()
    res.copy_(step(xx, dd).float().sum().view(1), non_blocking=True)
run("prefetch + d2h", pref)
def pref2():
    xx, dd = pf.get()
    pf.prefetch()
    step(xx, dd)
run("prefetch, no d2h", pref2)
