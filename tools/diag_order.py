"""Diagnostic: eager vs graph step time, alternating order (not collected)."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops
from paper_2407_04656_b200.graphs import GraphedStep
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
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
for _ in range(3):
    eager()
g = GraphedStep(layer, Tn, nbuf=1)
g.x[0].copy_(x); g.dout[0].copy_(dout)
def timeit(fn, n=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
for rnd in range(3):
    te = timeit(eager)
    tg = timeit(lambda: g.replay(0))
    tg2 = timeit(lambda: g.replay(0))
    te2 = timeit(eager)
    print(f"round {rnd}: eager {te:.3f}  graph {tg:.3f}  graph {tg2:.3f}  eager {te2:.3f}", flush=True)
