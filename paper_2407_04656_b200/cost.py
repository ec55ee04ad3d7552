"""The reference's time model of this path, evaluated on the device plan (SURVEY.md 8a
row a12; flexep simulator.py:198-266).

    adaptive_layer_cost(plan, layer_tokens, n_ranks) -> (max_node_tokens, cross_tokens)
        simulator.py:198-219: T split uniformly over the ranks (split_proportionally
        with unit weights), D = full_dispatch_matrices(T, R) -- here the bit-exact
        device planner (lz_plan_matrices) -- then the per-node received tokens and the
        tokens that cross a node boundary.
    step_time_model(plans, layer_loads, cost_model, n_ranks)      simulator.py:248-266
        (the "adaptive" strategy): overhead + sum_l alpha max_node_l + beta cross_l.
    plan_cost(D)
        the same two numbers for any device plan D [N, E, N] (e.g. a layer's last plan
        on its real routing: ``MoELayer.layer_cost``), two reductions on the device.
"""

from __future__ import annotations

from typing import Sequence

import torch

from . import _lib
from .dispatch import ReplicaMatrix, _dev, _raise_err


def plan_cost(D: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(max over nodes of received tokens, tokens sent off-node) of D [N, E, N] as device
    int64 scalars (no sync)."""
    recv = D.sum(dim=(0, 1), dtype=torch.int64)
    per_ij = D.sum(dim=1, dtype=torch.int64)
    return recv.max(), per_ij.sum() - per_ij.diagonal().sum()


def _uniform_T(layer_tokens: Sequence[int], n_ranks: int) -> list[list[int]]:
    # split_proportionally(t, [1] * n) (core.py:321-341): equal remainders, so the
    # leftover goes to the lowest indices
    out = []
    for t in layer_tokens:
        q, r = divmod(int(t), n_ranks)
        out.append([q + (1 if j < r else 0) for j in range(n_ranks)])
    return out


def adaptive_layer_cost(plan, layer_tokens: Sequence[int], n_ranks: int) -> tuple[int, int]:
    """Drop-in for flexep.simulator.adaptive_layer_cost (simulator.py:198-219). ``plan``
    is a placement plan (``column(j)``) or a ReplicaMatrix / E x N counts."""
    if isinstance(plan, ReplicaMatrix):
        R = plan.counts
    elif hasattr(plan, "column"):
        R = ReplicaMatrix.from_plan(plan).counts
    else:
        R = plan
    dev = _dev()
    E = len(layer_tokens)
    Tt = torch.tensor(_uniform_T(layer_tokens, n_ranks), dtype=torch.int32, device=dev)
    Rt = torch.tensor([list(r) for r in R], dtype=torch.int32, device=dev)
    D = torch.empty((n_ranks, E, n_ranks), dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("lz_plan_matrices", _lib.ptr(Tt), _lib.ptr(Rt), E, n_ranks, None, _lib.ptr(D),
              _lib.ptr(err), _lib.stream_ptr())
    mx, cross = plan_cost(D)
    vals = torch.stack([mx, cross, err[0].to(torch.int64)]).tolist()
    _raise_err(int(vals[2]))
    return int(vals[0]), int(vals[1])


def step_time_model(plans: dict, layer_loads: dict, cost_model, n_ranks: int) -> float:
    """flexep.simulator.step_time_model for the adaptive strategy (simulator.py:248-266);
    ``cost_model`` has per_token_compute_s, per_token_comm_s, step_overhead_s."""
    total = cost_model.step_overhead_s
    for layer, tokens in sorted(layer_loads.items()):
        max_node, cross = adaptive_layer_cost(plans[layer], tokens, n_ranks)
        total += cost_model.per_token_compute_s * max_node + cost_model.per_token_comm_s * cross
    return total


__all__ = ["adaptive_layer_cost", "plan_cost", "step_time_model"]
