"""Same-process A/B of a layer switch over the whole graphed fwd+bwd step, at any N:
two CUDA graphs (attribute off / on), replayed in alternating blocks so power / thermal
drift hits both arms alike; per-block times are the max over ranks.

    python tools/step_ab.py --attr tail_overlap [--config cfg2] [--blocks 8]
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/step_ab.py --attr early_router_wgrad
"""

from __future__ import annotations

import argparse
import math
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402
from paper_2407_04656_b200 import ops  # noqa: E402
from paper_2407_04656_b200.graphs import GraphedStep  # noqa: E402
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--attr", required=True)
    ap.add_argument("--values", default="0,1",
                    help="the two values of the attribute (ints; 0/1 = off/on for switches)")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    cfg = CONFIGS[a.config]
    E, k, d, dff, Tn = cfg["E"], cfg["k"], cfg["d"], cfg["dff"], cfg["tokens"]
    bias = zipf_router_bias(E, cfg["s"], seed=0)
    loads = (torch.softmax(bias, 0) * Tn * world * k).round().long().clamp_min(1).tolist()
    R = replica_matrix(plan_for_loads(loads, world, math.ceil(cfg["slot_factor"] * E / world), 2))
    layer = MoELayer(d, dff, E, k, seed=0, router_bias=bias, device=dev, replicas=R,
                     group=group, activation=cfg.get("act", "gelu"),
                     router_std=1.28 / math.sqrt(d))
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(Tn, d, generator=g, device=dev).bfloat16()
    dout = (torch.randn(Tn, d, generator=g, device=dev) * 1e-2).bfloat16()
    vals = [int(v) for v in a.values.split(",")]
    cur = getattr(layer, a.attr)
    conv = (lambda v: bool(v)) if cur is None or isinstance(cur, bool) else int
    graphs = {}
    for flag in (False, True):
        setattr(layer, a.attr, conv(vals[int(flag)]))
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
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.steps):
                graphs[flag].replay(0)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / a.steps], device=dev)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms[flag].append(float(t))
    if rank == 0:
        for flag in (False, True):
            print(f"N={world} {a.config} {a.attr}={vals[int(flag)]}: median "
                  f"{statistics.median(ms[flag]):.4f} ms/step  {[round(v, 3) for v in ms[flag]]}")
        print(f"parameter gradients bit-identical: {same}", flush=True)
    if world > 1:
        dist.barrier()
    # skip the interpreter teardown of two captured multi-rank graphs (NCCL + symmetric
    # memory): it can outlive the results by minutes
    sys.stdout.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
