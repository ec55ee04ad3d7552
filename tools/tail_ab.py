"""Same-process A/B of the backward tail overlap (layer.tail_overlap) at cfg2, N = 1:
two CUDA graphs of the whole fwd+bwd step (off / on), replayed in alternating blocks so
power / thermal drift hits both arms alike.  python tools/tail_ab.py [--blocks 8]"""

from __future__ import annotations

import argparse
import math
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402
from paper_2407_04656_b200 import ops  # noqa: E402
from paper_2407_04656_b200.graphs import GraphedStep  # noqa: E402
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    cfg = CONFIGS["cfg2"]
    E, k, d, dff, Tn = cfg["E"], cfg["k"], cfg["d"], cfg["dff"], cfg["tokens"]
    dev = torch.device("cuda", 0)
    layer = MoELayer(d, dff, E, k, seed=0, router_bias=zipf_router_bias(E, cfg["s"], seed=0),
                     device=dev, router_std=1.28 / math.sqrt(d))
    g = torch.Generator(device=dev).manual_seed(1234)
    x = torch.randn(Tn, d, generator=g, device=dev).bfloat16()
    dout = (torch.randn(Tn, d, generator=g, device=dev) * 1e-2).bfloat16()
    hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
    layer.set_plan(replica_matrix(plan_for_loads(hist.cpu().tolist(), 1,
                                                 math.ceil(cfg["slot_factor"] * E), 2)))
    graphs = {}
    for flag in (False, True):
        layer.tail_overlap = flag
        gs = GraphedStep(layer, Tn, nbuf=1, backward=True)
        gs.x[0].copy_(x)
        gs.dout[0].copy_(dout)
        graphs[flag] = gs
    grads = {}
    for flag, gs in graphs.items():
        gs.replay(0)
        torch.cuda.synchronize()
        grads[flag] = [p.grad.clone() for p in gs.params]
    same = all(torch.equal(u, v) for u, v in zip(grads[False], grads[True]))
    for gs in graphs.values():
        for _ in range(5):
            gs.replay(0)
    torch.cuda.synchronize()
    ms = {False: [], True: []}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for b in range(a.blocks):
        for flag in ((False, True) if b % 2 == 0 else (True, False)):
            e0.record()
            for _ in range(a.steps):
                graphs[flag].replay(0)
            e1.record()
            torch.cuda.synchronize()
            ms[flag].append(e0.elapsed_time(e1) / a.steps)
    for flag in (False, True):
        print(f"tail_overlap={int(flag)}: median {statistics.median(ms[flag]):.4f} ms/step  "
              f"{[round(v, 3) for v in ms[flag]]}")
    print(f"parameter gradients bit-identical: {same}")


if __name__ == "__main__":
    main()
