"""Multi-rank MoE layer check (run under torchrun, one rank per GPU, NCCL):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dist_layer_check.py [--elastic] [--rebalance]

Every rank routes its own tokens through the flexible all-to-all; outputs, input
grads and the replica-group-summed expert grads are compared with the torch-CPU
fp32 oracle evaluated on the gathered global batch (tolerances as in
tests/test_layer_gpu.py).  With --elastic, ranks are then removed (8 -> 6 -> 4 style:
the highest ranks leave), the host re-plans over the survivors with the reference
recipe, and the same kernels run the new plan.  Prints "DIST OK" on success.
"""

from __future__ import annotations

import math
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import moe_ref  # noqa: E402
from paper_2407_04656_b200 import ops  # noqa: E402
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402


def rel(got, ref):
    got, ref = got.detach().float().cpu(), ref.detach().float().cpu()
    return float((got - ref).norm() / ref.norm().clamp_min(1e-12))


def _gather_rows(t, group, sizes):
    """all-gather of per-rank row blocks of different lengths (padded to the max)."""
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    out = [torch.empty_like(pad) for _ in sizes]
    dist.all_gather(out, pad, group=group)
    return [o[:sz] for o, sz in zip(out, sizes)]


def check(layer, group, Tn, seed, tag, ragged=False):
    """ragged: every rank routes a different number of tokens (Tn + 96 * rank) -- the
    reference allows arbitrary per-rank counts T[e][j]."""
    rank, n = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev)
    g.manual_seed(seed + rank)
    sizes = [Tn + (96 * r if ragged else 0) for r in range(n)]
    Tn = sizes[rank]
    x = torch.randn(Tn, layer.d, generator=g, device=dev).bfloat16().requires_grad_(True)
    dout = torch.randn(Tn, layer.d, generator=g, device=dev).bfloat16()
    from paper_2407_04656_b200.layer import run_step

    def step():
        layer.zero_grad(set_to_none=True)
        x.grad = None
        o = layer(x)
        o.backward(dout)
        return o

    out = run_step([layer], step)   # grows the exchange buffers if the plan needs it
    k, E = layer.k, layer.E
    gidx = ops.router_gate(x.detach(), layer.wg.detach(), layer.bg.detach(), k)[0]
    # gather the global batch on every rank
    xs = _gather_rows(x.detach().contiguous(), group, sizes)
    ds = _gather_rows(dout, group, sizes)
    ids = _gather_rows(gidx, group, sizes)
    # full weights: every owner holds the deterministic per-expert init (no optimizer step)
    from paper_2407_04656_b200.layer import _expert_weights
    w1 = torch.stack([_expert_weights(layer.seed, 2 * e, (layer.d_ff, layer.d), layer.init_std, dev)
                      for e in range(E)]).float().cpu().requires_grad_(True)
    w2 = torch.stack([_expert_weights(layer.seed, 2 * e + 1, (layer.d, layer.d_ff), layer.init_std,
                                      dev) for e in range(E)]).float().cpu().requires_grad_(True)
    for p, e in enumerate(layer.local_ids):
        assert torch.equal(layer.w1.detach()[p].float().cpu(), w1.detach()[e]), f"expert {e} copy"
    X = torch.cat([t.float().cpu() for t in xs]).requires_grad_(True)
    wg = layer.wg.detach().float().cpu().requires_grad_(True)
    bg = layer.bg.detach().float().cpu().requires_grad_(True)
    ref, _, _, _ = moe_ref.moe_forward_ref(X, wg, bg, w1, w2, k, layer.renorm,
                                           idx=torch.cat([t.cpu() for t in ids]))
    ref.backward(torch.cat([t.float().cpu() for t in ds]))
    sl = slice(sum(sizes[:rank]), sum(sizes[:rank + 1]))
    errs = {"out": rel(out, ref[sl]), "dx": rel(x.grad, X.grad[sl]), "dwg": rel(layer.wg.grad, wg.grad),
            "dbg": rel(layer.bg.grad, bg.grad)}
    for p, e in enumerate(layer.local_ids):
        errs[f"dW1[{e}]"] = rel(layer.w1.grad[p], w1.grad[e])
        errs[f"dW2[{e}]"] = rel(layer.w2.grad[p], w2.grad[e])
    bad = {kk: v for kk, v in errs.items() if v > (5e-2 if kk in ("dwg", "dbg") else 3e-2)}
    print(f"[{tag}] rank {rank}/{n} local experts {layer.local_ids} imbalance "
          f"{layer.imbalance():.3f} max rel err {max(errs.values()):.3e}", flush=True)
    assert not bad, f"rank {rank}: {bad}"


def multilayer(group, n_layers=4):
    """A stack of cfg2-sized layers (E16 top-2, d1024, d_ff4096, 65,536 tokens per rank):
    the plan-sized exchange buffers (1.25 x the balanced share, not N x Tn x k) keep a
    multi-layer step within HBM; one fwd + bwd through all layers, peak memory reported."""
    n = dist.get_world_size(group)
    E, k, d, dff, Tn = 16, 2, 1024, 4096, 65536
    bias = zipf_router_bias(E, 1.2, seed=0)
    loads = (torch.softmax(bias, 0) * Tn * n * k).round().long().clamp_min(1).tolist()
    R = replica_matrix(plan_for_loads(loads, n, math.ceil(6 * E / n), 2))
    layers = [MoELayer(d, dff, E, k, replicas=R, group=group, seed=li, router_bias=bias,
                       router_std=1.28 / math.sqrt(d)) for li in range(n_layers)]
    torch.cuda.reset_peak_memory_stats()
    g = torch.Generator(device="cuda")
    g.manual_seed(dist.get_rank(group))
    x = torch.randn(Tn, d, generator=g, device="cuda").bfloat16().requires_grad_(True)
    from paper_2407_04656_b200.layer import run_step
    runs = []

    def step():
        runs.append(1)
        x.grad = None
        h = x
        for L in layers:
            h = h + L(h)          # residual stream, as in a transformer block
        h.float().square().mean().backward()
        return h

    h = run_step(layers, step)
    retries = len(runs) - 1
    peak = torch.cuda.max_memory_allocated() / 2**30
    # symmetric exchange buffers exist only with the P2P exchange (LZ_EXCHANGE=nccl: none)
    rows = [L._symm.rows if L._symm is not None else None for L in layers]
    print(f"[{n_layers} layers N={n}] rank {dist.get_rank(group)} exchange rows {rows} "
          f"(N*Tn*k = {n * Tn * k}), capacity re-runs {retries}, peak memory {peak:.1f} GiB",
          flush=True)
    assert torch.isfinite(x.grad.float()).all()
    del layers, h, x


def kill_mid_step(layer, group, Tn, loads, c):
    """A rank dies mid-step -- after the histogram all-gather and its dispatch, before
    its expert GEMMs and the combine.  The survivors' device waits (arrival
    flags, peer barrier) give up after the control block's timeout instead of hanging,
    check() raises StepAbortedError, the step is discarded, and the survivors shrink the
    communicator, re-plan with the reference recipe, move the expert state and resume."""
    from paper_2407_04656_b200 import _lib, comm
    from paper_2407_04656_b200.elastic import shrink_and_replan
    from paper_2407_04656_b200.layer import StepAbortedError
    cur = dist.get_world_size(group)
    me = dist.get_rank(group)
    victim = cur - 1
    _lib.control(timeout_s=3.0)
    _lib.control_reset()
    dist.barrier(group=group)
    torch.cuda.synchronize()

    class Dying(comm.ProcessFabric):
        def serve(self, req):
            if req[0] == comm.SYNC:          # after this rank's dispatch + arrival signal
                torch.cuda.synchronize()
                print(f"rank {dist.get_rank()} dies mid-step", flush=True)
                os._exit(0)
            return super().serve(req)

    if me == victim:
        fab = Dying(group)
        layer.fabric = fab
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.randn(Tn, layer.d, generator=g, device="cuda").bfloat16()
    with torch.no_grad():
        layer(x)
    torch.cuda.synchronize()
    try:
        layer.check()
        raise AssertionError("a lost peer must abort the step")
    except StepAbortedError as exc:
        print(f"rank {dist.get_rank()} step aborted: {exc.status}", flush=True)
    _lib.control_reset()
    _lib.control(timeout_s=10.0)
    opt = torch.optim.Adam([layer.w1, layer.w2], lr=1e-4)
    # the survivors need slots for every expert (f_eff drops with the node count)
    slots = max(c, math.ceil(layer.E / (cur - 1)))
    layer, group, rep = shrink_and_replan(layer, group, [victim], loads, slots, optimizer=opt)
    if dist.get_rank(group) == 0:
        print(f"re-plan after mid-step loss: {rep}", flush=True)
    check(layer, group, Tn, 400, f"N={dist.get_world_size(group)} after mid-step loss")
    return layer, group


def main():
    elastic = "--elastic" in sys.argv
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, n = dist.get_rank(), dist.get_world_size()
    E, k, d, dff, Tn = 8, 2, 512, 1024, 2048
    bias = zipf_router_bias(E, 1.2, seed=2)
    loads = (torch.softmax(bias, 0) * Tn * n * k).round().long().clamp_min(1).tolist()
    c = math.ceil(3 * E / n)
    R = replica_matrix(plan_for_loads(loads, n, c, 2))
    layer = MoELayer(d, dff, E, k, replicas=R, group=dist.group.WORLD, seed=7, init_std=0.05,
                     router_bias=bias)
    check(layer, dist.group.WORLD, Tn, 100, f"N={n}")
    check(layer, dist.group.WORLD, Tn, 150, f"N={n} ragged batches", ragged=True)
    group = dist.group.WORLD
    if "--rebalance" in sys.argv:
        # the routing skew moves (new hot experts): the device load window sees it and the
        # periodic rebalance re-places replicas, migrating expert weights over NVLink
        from paper_2407_04656_b200.rebalance import Rebalancer
        rb = Rebalancer([layer], c, 2, interval=3)
        layer.bg.data.copy_(zipf_router_bias(E, 2.0, seed=11).to(layer.bg.device))
        g = torch.Generator(device="cuda")
        g.manual_seed(rank)
        rep = None
        with torch.no_grad():
            for _ in range(3):
                layer(torch.randn(Tn, d, generator=g, device="cuda").bfloat16())
                rep = rb.step() or rep
        assert rep is not None and rep["changed"], rep
        if rank == 0:
            print(f"rebalance: {rep}", flush=True)
        check(layer, group, Tn, 300, f"N={n} after rebalance")
    if elastic and n > 2:
        from paper_2407_04656_b200.elastic import shrink_and_replan
        # 8 -> 6 -> 4 when launched on 8 GPUs (4 -> 3 -> 2 on 4): drop two ranks, twice
        step = max(1, n // 4)
        for _ in range(2):
            cur = dist.get_world_size(group)
            if cur - step < 2:
                break
            exclude = list(range(cur - step, cur))
            if dist.get_rank(group) in exclude:
                print(f"rank {rank} leaves (simulated failure)", flush=True)
                os._exit(0)
            # lr = 0: Adam's moments are populated from the last check's gradients while
            # the weights keep their deterministic values (check() rebuilds them)
            opt = torch.optim.Adam([layer.w1, layer.w2], lr=0.0)
            opt.step()
            layer, group, rep = shrink_and_replan(layer, group, exclude, loads, c, optimizer=opt)
            assert opt.param_groups[0]["params"][0] is layer.w1
            assert rep["optimizer_state_keys"] == ["exp_avg", "exp_avg_sq"], rep
            assert opt.state[layer.w1]["exp_avg"].shape[0] == len(layer.local_ids)
            if dist.get_rank(group) == 0:
                print(f"re-plan: {rep}", flush=True)
            check(layer, group, Tn, 200 + cur, f"N={dist.get_world_size(group)} after failure")
    if "--multilayer" in sys.argv:
        multilayer(group)
    if "--kill" in sys.argv and dist.get_world_size(group) >= 2:
        layer, group = kill_mid_step(layer, group, Tn, loads, c)
    dist.barrier(group=group)
    if dist.get_rank(group) == 0:
        print("DIST OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
