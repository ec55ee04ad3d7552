"""Diagnostic (torchrun): e2e step time variants at N ranks.  Not collected by pytest."""

import math
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2407_04656_b200 import ops  # noqa: E402
from paper_2407_04656_b200.hostio import HostPrefetcher  # noqa: E402
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    E, k, d, dff, Tn = 16, 2, 1024, 4096, 65536
    bias = zipf_router_bias(E, 1.2)
    layer = MoELayer(d, dff, E, k, router_bias=bias, device=dev, group=dist.group.WORLD)
    g = torch.Generator(device=dev)
    g.manual_seed(rank)
    x = torch.randn(Tn, d, generator=g, device=dev).bfloat16()
    dout = (torch.randn(Tn, d, generator=g, device=dev) * 1e-2).bfloat16()
    hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
    dist.all_reduce(hist)
    layer.set_plan(replica_matrix(plan_for_loads(hist.tolist(), n, math.ceil(3 * E / n), 2)))
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
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(K):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / K
        if rank == 0:
            print(f"{name:40s} {dt * 1e3:8.2f} ms/step", flush=True)

    run("resident", lambda: step(x, dout))
    run("h2d blocking copies", lambda: step(x_h.to(dev), d_h.to(dev)))
    run("h2d non_blocking", lambda: step(x_h.to(dev, non_blocking=True),
                                         d_h.to(dev, non_blocking=True)))

    def with_d2h():
        out = step(x_h.to(dev, non_blocking=True), d_h.to(dev, non_blocking=True))
        res.copy_(out.float().sum().view(1), non_blocking=True)
    run("h2d + d2h scalar", with_d2h)
    pf = HostPrefetcher([x_h, d_h], dev)
    pf.prefetch()

    def pref():
        xx, dd = pf.get()
        pf.prefetch()
        out = step(xx, dd)
        res.copy_(out.float().sum().view(1), non_blocking=True)
    run("prefetch", pref)
    pf.get()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
