"""Kernel timeline of the graphed cfg2 step at full clocks (torch.profiler / CUPTI):
per-kernel durations and the idle gaps between consecutive kernels of one replay.

    python tools/timeline.py [--config cfg2] [--reps 5]
"""

from __future__ import annotations

import argparse
import collections
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import CONFIGS  # noqa: E402
from paper_2407_04656_b200 import ops  # noqa: E402
from paper_2407_04656_b200.graphs import GraphedStep  # noqa: E402
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    E, k, d, dff, Tn = cfg["E"], cfg["k"], cfg["d"], cfg["dff"], cfg["tokens"]
    layer = MoELayer(d, dff, E, k, seed=0, router_bias=zipf_router_bias(E, cfg["s"], seed=0),
                     activation=cfg.get("act", "gelu"), router_std=1.28 / math.sqrt(d))
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    x = torch.randn(Tn, d, generator=g, device="cuda").bfloat16()
    dout = (torch.randn(Tn, d, generator=g, device="cuda") * 1e-2).bfloat16()
    hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3]
    layer.set_plan(replica_matrix(plan_for_loads(hist.long().cpu().tolist(), 1,
                                                 math.ceil(cfg["slot_factor"] * E), 2)))
    gs = GraphedStep(layer, Tn, nbuf=1)
    gs.x[0].copy_(x)
    gs.dout[0].copy_(dout)
    for _ in range(5):
        gs.replay(0)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            gs.replay(0)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    ev.sort(key=lambda e: e.time_range.start)
    # split into replays at gaps > 50 us? use the kernel count per replay instead
    n = len(ev) // a.reps
    per = collections.defaultdict(list)
    gaps = collections.defaultdict(list)
    steps = []
    for r in range(a.reps):
        seq = ev[r * n:(r + 1) * n]
        steps.append(seq[-1].time_range.end - seq[0].time_range.start)
        for i, e in enumerate(seq):
            per[(i, e.name[:60])].append(e.time_range.elapsed_us())
            if i:
                gaps[(i, e.name[:60])].append(e.time_range.start - seq[i - 1].time_range.end)
    tot_k = tot_g = 0.0
    print(f"{'#':>3} {'kernel':60s} {'us':>8} {'gap_before':>10}")
    for (i, name), v in sorted(per.items()):
        m = sorted(v)[len(v) // 2]
        gp = sorted(gaps.get((i, name), [0.0]))[len(gaps.get((i, name), [0.0])) // 2]
        tot_k += m
        tot_g += gp
        print(f"{i:3d} {name:60s} {m:8.1f} {gp:10.1f}")
    print(f"kernels {tot_k:.1f} us, gaps {tot_g:.1f} us, step (first start..last end) "
          f"{sorted(steps)[len(steps) // 2]:.1f} us, {n} kernels per replay")


if __name__ == "__main__":
    main()
