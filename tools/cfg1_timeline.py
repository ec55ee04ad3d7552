"""Kernel timeline of the graphed cfg1 (4 virtual ranks) forward."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2407_04656_b200.layer import zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402
from paper_2407_04656_b200.virtual import VirtualEP  # noqa: E402

cfg = CONFIGS["cfg1"]
nv, Tn, E, k, d, dff = 4, cfg["tokens"], cfg["E"], cfg["k"], cfg["d"], cfg["dff"]
bias = zipf_router_bias(E, cfg["s"])
p = torch.softmax(bias, 0).tolist()
loads = [max(1, int(v * Tn * nv * k)) for v in p]
R = replica_matrix(plan_for_loads(loads, nv, math.ceil(cfg["slot_factor"] * E / nv), 2))
vep = VirtualEP(d, dff, E, k, R, Tn, seed=0, router_bias=bias)
xs = [torch.randn(Tn, d, device="cuda").bfloat16() for _ in range(nv)]
for _ in range(3):
    vep(xs)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    vep(xs)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.replay()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.elapsed_us():7.1f}  {e.name[:70]}")
print("span", ev[-1].time_range.end - t0)
