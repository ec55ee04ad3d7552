"""Where does the e2e (host-input) step lose time vs the device-resident replay?
cfg2 at N = 1:  python tools/e2e_probe.py"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops  # noqa: E402
from paper_2407_04656_b200.graphs import GraphedStep  # noqa: E402
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402

E, k, d, dff, Tn = 16, 2, 1024, 4096, 65536
dev = torch.device("cuda")
layer = MoELayer(d, dff, E, k, seed=0, router_bias=zipf_router_bias(E, 1.2, seed=0), device=dev,
                 router_std=1.28 / math.sqrt(d))
g = torch.Generator(device=dev).manual_seed(1234)
x = torch.randn(Tn, d, generator=g, device=dev).bfloat16()
dout = (torch.randn(Tn, d, generator=g, device=dev) * 1e-2).bfloat16()
hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
layer.set_plan(replica_matrix(plan_for_loads(hist.cpu().tolist(), 1, 80, 2)))
gs = GraphedStep(layer, Tn, nbuf=2)
for b in range(2):
    gs.x[b].copy_(x)
    gs.dout[b].copy_(dout)
x_h, d_h = x.cpu().pin_memory(), dout.cpu().pin_memory()
res_h = torch.empty(1).pin_memory()
cs = torch.cuda.Stream()
main = torch.cuda.current_stream()
ev_copy = [torch.cuda.Event() for _ in range(2)]
ev_done = [torch.cuda.Event() for _ in range(2)]


def run(n, copies, alternate, readback):
    for b in range(2):
        ev_done[b].record(main)

    def h2d(b):
        with torch.cuda.stream(cs):
            cs.wait_event(ev_done[b])
            if copies:
                gs.x[b].copy_(x_h, non_blocking=True)
                gs.dout[b].copy_(d_h, non_blocking=True)
            ev_copy[b].record(cs)

    h2d(0)
    for i in range(n):
        b = i % 2 if alternate else 0
        main.wait_event(ev_copy[b])
        r = gs.replay(b)
        ev_done[b].record(main)
        if readback:
            res_h.copy_(r, non_blocking=True)
        if i + 1 < n:
            h2d((i + 1) % 2 if alternate else 0)


for name, kw in [("replay(0) only", dict(copies=False, alternate=False, readback=False)),
                 ("alternate buffers", dict(copies=False, alternate=True, readback=False)),
                 ("+ readback", dict(copies=False, alternate=True, readback=True)),
                 ("+ H2D copies (e2e)", dict(copies=True, alternate=True, readback=True)),
                 ("replay(0) only", dict(copies=False, alternate=False, readback=False))]:
    for n in (10, 30):
        run(3, **kw)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(n, **kw)
        b.record()
        torch.cuda.synchronize()
        print(f"{name:22s} n={n:2d}: {a.elapsed_time(b) / n:.3f} ms/step", flush=True)
