"""Elastic reconfiguration of the MoE layer after rank failures (BASELINE config 5).

Recipe of the reference controller (controller.py:392-451, simulator.py:363-384):
  1. the survivors form a new communicator (torch ``dist.shrink_group`` -> NCCL
     ncclCommShrink; excluded ranks take no part),
  2. the host re-plans for the live set: allocate_replicas + build_mro_plan with
     f_eff = min(f, N_live) (core.py:113), greedy_node_mapping of surviving nodes onto
     the new plan columns (migration.py:75-120) -> column -> node order,
  3. experts a node must newly host are fetched from surviving owners, sends spread
     over owners as in plan_state_transfers (migration.py:164-195) -- here as batched
     NCCL send/recv of the expert weights over NVLink instead of the reference's TCP
     blob fetch (agent.py:196-244),
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


def exchange_expert_state(layers, transfers, me: int, rank_of: dict, group) -> list[dict]:
    """Batched NCCL send/recv (one ``batch_isend_irecv``) of the expert weights in
    ``transfers`` = [((layer index, expert), src_node, dst_node)].  Returns, per layer,
    {expert: (w1, w2)} = this rank's kept experts plus the received ones."""
    keep = [layer.expert_state() for layer in layers]
    got: list[dict] = [dict(k) for k in keep]
    ops = []
    for (li, e), src, dst in transfers:
        layer = layers[li]
        if src == me:
            w1, w2 = keep[li][e]
            ops.append(dist.P2POp(dist.isend, w1.contiguous(), rank_of[dst], group))
            ops.append(dist.P2POp(dist.isend, w2.contiguous(), rank_of[dst], group))
        elif dst == me:
            f1 = 2 * layer.d_ff if layer.activation == "swiglu" else layer.d_ff
            b1 = torch.empty((f1, layer.d), dtype=torch.bfloat16, device=layer.device)
            b2 = torch.empty((layer.d, layer.d_ff), dtype=torch.bfloat16, device=layer.device)
            ops.append(dist.P2POp(dist.irecv, b1, rank_of[src], group))
            ops.append(dist.P2POp(dist.irecv, b2, rank_of[src], group))
            got[li][e] = (b1, b2)
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    torch.cuda.synchronize()
    return got


def shrink_and_replan(layer, group, exclude: Sequence[int], loads: Sequence[int], slots: int,
                      fault_threshold: int = 2):
    """Remove ``exclude`` (ranks of ``group``) and move ``layer`` onto the survivors.
    Excluded ranks must not call this (they are gone); survivors all call it.
    Returns (layer, new_group, report)."""
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
    weights = exchange_expert_state([layer], [((0, e), src, dst) for e, src, dst in transfers],
                                    me, rank_of, new_group)[0]
    layer.group = new_group
    layer.rank = dist.get_rank(new_group)
    layer.world = dist.get_world_size(new_group)
    layer.node_ids = new_nodes
    layer.set_plan(R, weights=weights)
    report = {"live": new_nodes, "order": order, "transfers": len(transfers),
              "bytes": len(transfers) * 2 * layer.d * layer.d_ff * 2,
              "checkpoint_fallback": orphans, "replicas": list(plan.replica_counts)}
    return layer, new_group, report
