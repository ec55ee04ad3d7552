"""Elastic reconfiguration of the MoE layer after rank failures (BASELINE config 5).

Recipe of the reference controller (controller.py:392-451, simulator.py:363-384):
  1. the survivors form a new communicator (torch ``dist.shrink_group`` -> NCCL
     ncclCommShrink; excluded ranks take no part),
  2. the host re-plans for the live set: allocate_replicas + build_mro_plan with
     f_eff = min(f, N_live) (core.py:113), greedy_node_mapping of surviving nodes onto
     the new plan columns (migration.py:75-120) -> column -> node order,
  3. experts a node must newly host are fetched from surviving owners, sends spread
     over owners as in plan_state_transfers (migration.py:164-195) -- here as batched
     NCCL send/recv over NVLink of the expert weights AND their optimizer state
     ("weights and optimizer states") instead of the reference's TCP blob
     fetch (agent.py:196-244); the optimizer is re-pointed at the new parameters,
  4. the new replica matrix (communicator-rank order) is uploaded; the same kernels
     consume it without recompiling.
An expert without a surviving owner is re-initialised and reported, the analogue of
the reference's ``checkpoint_fallback`` event (controller.py:437-440).
"""

from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist

from .placement import (ClusterSpec, allocate_replicas, build_mro_plan, greedy_node_mapping,
                        node_order, plan_state_transfers, replica_matrix)


def replan(loads: Sequence[int], live_nodes: Sequence[int], holdings: dict, slots: int,
           fault_threshold: int = 2):
    """Host re-plan over ``live_nodes`` (node ids).  Returns (plan, order, R) where
    order[col] = node and R is in communicator-rank order (ranks = live nodes sorted)."""
    live = sorted(live_nodes)
    spec = ClusterSpec(len(live), slots, min(fault_threshold, len(live)))
    plan = build_mro_plan(allocate_replicas(loads, spec), spec)
    cols = [set(plan.column(j)) for j in range(plan.n_nodes)]
    assignment = greedy_node_mapping(holdings, cols, live)
    order = node_order(assignment)
    return plan, order, replica_matrix(plan, order)


def transfer_schedule(new_R, new_nodes: Sequence[int], holdings: dict):
    """[(expert, src_node, dst_node)] for experts a node must newly host; the source
    is the surviving owner with the fewest sends of that expert, then fewest sends
    overall, then the lowest node id (plan_state_transfers, migration.py:164-195).
    Experts with no surviving owner are returned separately (checkpoint fallback)."""
    fetch = {node: {e for e, row in enumerate(new_R) if row[r] > 0} - holdings.get(node, set())
             for r, node in enumerate(new_nodes)}
    owners: dict = {}
    for v in sorted(holdings):
        for e in holdings[v]:
            owners.setdefault(e, []).append(v)
    return plan_state_transfers(fetch, owners, allow_orphans=True)


def expert_slices(layer, optimizer=None, state_keys=None) -> dict:
    """{expert: [w1_e, w2_e, then every per-parameter optimizer state tensor of the same
    shape as its parameter, sliced to expert e]} -- the unit the reference migrates
    ("weights and optimizer states"; sized by state_size in
    migration.py:164-195).  ``state_keys`` (default: the tensor-valued, parameter-shaped
    entries of the optimizer's state of w1, e.g. Adam's exp_avg / exp_avg_sq)."""
    keys = list(state_keys) if state_keys is not None else optimizer_state_keys(layer, optimizer)
    out = {}
    for pos, e in enumerate(layer.local_ids):
        ts = [layer.w1.data[pos], layer.w2.data[pos]]
        for p in (layer.w1, layer.w2):
            st = optimizer.state.get(p, {}) if optimizer is not None else {}
            for key in keys:
                v = st.get(key)
                ts.append(v[pos] if v is not None else torch.zeros_like(p.data[pos]))
        out[e] = ts
    return out


def optimizer_state_keys(layer, optimizer) -> list:
    if optimizer is None:
        return []
    st = optimizer.state.get(layer.w1, {})
    return sorted(k for k, v in st.items()
                  if isinstance(v, torch.Tensor) and v.shape == layer.w1.shape)


def transfer_bytes(layer, n_state_keys: int = 0) -> int:
    """Bytes one migrated expert moves: its weight matrices (2 for GELU, W1|W3 + W2 for
    SwiGLU) and each per-parameter optimizer state of the same shapes."""
    w = layer.w1[0].numel() * layer.w1.element_size() + layer.w2[0].numel() * layer.w2.element_size()
    st = 0
    if n_state_keys:
        st = n_state_keys * (layer.w1[0].numel() + layer.w2[0].numel()) * 4
    return w + st


def exchange_expert_state(layers, transfers, me: int, rank_of: dict, group,
                          optimizers=None, state_keys=None) -> list[dict]:
    """Batched NCCL send/recv (one ``batch_isend_irecv``) of the expert state in
    ``transfers`` = [((layer index, expert), src_node, dst_node)]: weights and, with
    ``optimizers`` (one per layer, or None), the per-expert optimizer state.  Returns, per
    layer, {expert: [w1, w2, *states]} = this rank's kept experts plus the received ones
    (feed ``[0:2]`` to ``set_plan`` and the rest to :func:`remap_optimizer`)."""
    optimizers = optimizers or [None] * len(layers)
    keys = [list(state_keys) if state_keys is not None else optimizer_state_keys(L, o)
            for L, o in zip(layers, optimizers)]
    keep = [expert_slices(L, o, k) for L, o, k in zip(layers, optimizers, keys)]
    got: list[dict] = [dict(k) for k in keep]
    ops = []
    for (li, e), src, dst in transfers:
        layer = layers[li]
        if src == me:
            for t in keep[li][e]:
                ops.append(dist.P2POp(dist.isend, t.contiguous(), rank_of[dst], group))
        elif dst == me:
            f1 = 2 * layer.d_ff if layer.activation == "swiglu" else layer.d_ff
            shapes = [((f1, layer.d), torch.bfloat16), ((layer.d, layer.d_ff), torch.bfloat16)]
            for i in range(2):
                st = optimizers[li].state.get((layer.w1, layer.w2)[i], {}) if optimizers[li] else {}
                for key in keys[li]:
                    v = st.get(key)
                    dt = v.dtype if v is not None else torch.float32
                    shapes.append((shapes[i][0], dt))
            bufs = [torch.empty(shp, dtype=dt, device=layer.device) for shp, dt in shapes]
            for b in bufs:
                ops.append(dist.P2POp(dist.irecv, b, rank_of[src], group))
            got[li][e] = bufs
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if layers and layers[0].device.type == "cuda":
        torch.cuda.synchronize()
    return got


def remap_optimizer(optimizer, layer, info: dict, slices: dict, state_keys=None) -> None:
    """After ``layer.set_plan`` replaced w1/w2 (``info`` = its return value): swap the
    new Parameters into ``optimizer``'s param groups and rebuild their per-expert state
    from ``slices`` ({expert: [w1, w2, *states]} of exchange_expert_state; experts
    missing from it -- checkpoint fallback -- start from zero state).  Scalar state
    entries (Adam's step) carry over."""
    old_w1, old_w2 = info["replaced"]
    new_w1, new_w2 = info["params"]
    keys = list(state_keys) if state_keys is not None else \
        sorted(k for k, v in optimizer.state.get(old_w1, {}).items()
               if isinstance(v, torch.Tensor) and old_w1 is not None and v.shape == old_w1.shape)
    for group in optimizer.param_groups:
        group["params"] = [new_w1 if p is old_w1 else new_w2 if p is old_w2 else p
                           for p in group["params"]]
    for i, (old, new) in enumerate(((old_w1, new_w1), (old_w2, new_w2))):
        st_old = optimizer.state.pop(old, {}) if old is not None else {}
        if not st_old:
            continue
        st_new = {k: v for k, v in st_old.items() if k not in keys}
        for j, key in enumerate(keys):
            per = []
            for e in info["local_ids"]:
                src = slices.get(e)
                t = src[2 + i * len(keys) + j] if src is not None and len(src) > 2 else None
                per.append(t.to(st_old[key].dtype) if t is not None
                           else torch.zeros_like(new.data[0], dtype=st_old[key].dtype))
            st_new[key] = torch.stack(per).contiguous()
        optimizer.state[new] = st_new


def shrink_and_replan(layer, group, exclude: Sequence[int], loads: Sequence[int], slots: int,
                      fault_threshold: int = 2, optimizer=None):
    """Remove ``exclude`` (ranks of ``group``) and move ``layer`` onto the survivors.
    Excluded ranks must not call this (they are gone); survivors all call it.  With an
    ``optimizer`` the migrated experts' optimizer state moves with their weights and the
    optimizer is re-pointed at the new parameters.  Returns (layer, new_group, report)."""
    from .comm import ProcessFabric
    old_rank = dist.get_rank(group)
    if old_rank in exclude:
        raise RuntimeError("an excluded rank cannot take part in the shrink")
    nodes = getattr(layer, "node_ids", list(range(dist.get_world_size(group))))
    holdings = {nodes[j]: {e for e, row in enumerate(layer.R) if row[j] > 0}
                for j in range(len(nodes)) if j not in exclude}
    live = sorted(holdings)
    new_group = dist.shrink_group(list(exclude), group=group)
    plan, order, R = replan(loads, live, holdings, slots, fault_threshold)
    new_nodes = live  # communicator rank r <-> node live[r]
    me = nodes[old_rank]
    transfers, orphans = transfer_schedule(R, new_nodes, holdings)
    rank_of = {v: r for r, v in enumerate(new_nodes)}
    keys = optimizer_state_keys(layer, optimizer)
    slices = exchange_expert_state([layer], [((0, e), src, dst) for e, src, dst in transfers],
                                   me, rank_of, new_group, [optimizer], keys)[0]
    layer.set_fabric(ProcessFabric(new_group))
    layer.node_ids = new_nodes
    info = layer.set_plan(R, weights={e: (v[0], v[1]) for e, v in slices.items()})
    if optimizer is not None:
        remap_optimizer(optimizer, layer, info, slices, keys)
    report = {"live": new_nodes, "order": order, "transfers": len(transfers),
              "bytes": len(transfers) * transfer_bytes(layer, len(keys)),
              "optimizer_state_keys": keys,
              "checkpoint_fallback": orphans, "replicas": list(plan.replica_counts)}
    return layer, new_group, report
