"""Diagnostic: CUDA-graph capture of the multi-rank (P2P exchange) step under torchrun.

    timeout 240 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/graph_dist.py [--fwd-only]
"""

from __future__ import annotations

import math
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2407_04656_b200 import ops  # noqa: E402
from paper_2407_04656_b200.graphs import GraphedStep  # noqa: E402
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402


def log(*a):
    print(f"[rank {dist.get_rank()} t={time.time() % 1000:.2f}]", *a, flush=True)


def main():
    fwd_only = "--fwd-only" in sys.argv
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    E, k, d, dff, Tn = 16, 2, 1024, 4096, 16384
    bias = zipf_router_bias(E, 1.2, seed=0)
    layer = MoELayer(d, dff, E, k, seed=0, router_bias=bias, device=dev,
                     router_std=1.28 / math.sqrt(d), group=dist.group.WORLD)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn(Tn, d, generator=g, device=dev).bfloat16()
    dout = (torch.randn(Tn, d, generator=g, device=dev) * 1e-2).bfloat16()
    hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
    dist.all_reduce(hist)
    layer.set_plan(replica_matrix(plan_for_loads(hist.cpu().tolist(), n, math.ceil(5 * E / n), 2)))
    for _ in range(3):
        layer.zero_grad(set_to_none=True)
        out = layer(x)
        if not fwd_only:
            out.backward(dout)
    torch.cuda.synchronize()
    ref = out.detach().clone()
    ref_g = None if fwd_only else layer.w1.grad.detach().clone()
    del out
    log("eager ok; capturing")
    dist.barrier()
    gs = GraphedStep(layer, Tn, nbuf=1, backward=not fwd_only)
    log("captured")
    gs.x[0].copy_(x)
    gs.dout[0].copy_(dout)
    dist.barrier()
    torch.cuda.synchronize()
    for _ in range(3):
        gs.replay(0)
    torch.cuda.synchronize()
    log("replayed")
    if not fwd_only:
        assert torch.equal(layer.w1.grad, ref_g), "dW1 differs from eager"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        gs.replay(0)
    e1.record()
    torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / 10
    dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        layer.zero_grad(set_to_none=True)
        out = layer(x)
        if not fwd_only:
            out.backward(dout)
    e1.record()
    torch.cuda.synchronize()
    t_eager = e0.elapsed_time(e1) / 10
    log(f"graph {t_graph:.3f} ms/step, eager {t_eager:.3f} ms/step")
    dist.barrier()
    if rank == 0:
        print("GRAPH DIST OK", flush=True)
    del gs
    torch.cuda.synchronize()
    log("graph released")
    dist.destroy_process_group()
    log("destroyed")


if __name__ == "__main__":
    main()
