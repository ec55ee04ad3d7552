"""Periodic load-driven rebalance of the replica placement.

The reference's adaptive strategy keeps a trailing window of per-step expert loads
(simulator.py:642-644, the controller's load reports controller.py:279-284) and every
``rebalance_interval_steps`` (core.py:55, default 200) re-allocates replicas from the
window's integer mean (simulator.py:342-351 ``window_loads``), re-places them with the
MRO placement, maps nodes onto the new columns with the greedy minimum-migration
mapping jointly over all layers' (layer, expert) items and moves the state
(simulator.py:363-384 ``rebuild_adaptive_plans``; controller.py:408-450).

B200 version:
  * the window lives on the device: every forward records the all-gathered load matrix's
    row sums into a ring (``lz_load_record``, one tiny launch, CUDA-graph safe);
  * every rank holds the identical T, hence identical loads and an identical new plan --
    no negotiation, as in the reference's dispatch (dispatch.py:132-135);
  * newly hosted experts are fetched from current owners over NVLink in one batched
    NCCL send/recv (``exchange_expert_state``); the kernels consume the new R without
    recompiling.
"""

from __future__ import annotations

from typing import Sequence

import torch

from . import _lib
from ._lib import ptr
from .placement import (ClusterSpec, allocate_replicas, build_mro_plan, greedy_node_mapping,
                        node_order, plan_state_transfers, replica_matrix)


class LoadWindow:
    """Device ring of the last ``window`` steps' global per-expert loads."""

    def __init__(self, n_experts: int, window: int = 200, device=None):
        self.E, self.W = n_experts, window
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.ring = torch.zeros((window, n_experts), dtype=torch.int64, device=dev)
        self.pos = torch.zeros(1, dtype=torch.int64, device=dev)

    def record(self, T: torch.Tensor) -> None:
        """T: int32 [E, N] all-gathered load matrix of one step (device)."""
        if T.dtype != torch.int32 or not T.is_contiguous() or T.shape[0] != self.E:
            raise ValueError("T must be a contiguous int32 [E, N] tensor")
        _lib.call("lz_load_record", ptr(T), self.E, T.shape[1], ptr(self.ring), self.W,
                  ptr(self.pos), torch.cuda.current_stream(T.device).cuda_stream)

    def steps(self) -> int:
        return int(self.pos.item())

    def loads(self) -> tuple[int, ...] | None:
        """Integer mean over the recorded window (simulator.py:342-351); None if empty.
        Host read (one sync) -- called at a rebalance only."""
        n = min(self.steps(), self.W)
        if n == 0:
            return None
        return tuple(int(v) for v in (self.ring[:n].sum(0) // n).tolist())

    def reset(self) -> None:
        self.ring.zero_()
        self.pos.zero_()


def plan_rebalance(R_layers: Sequence[Sequence[Sequence[int]]], node_ids: Sequence[int],
                   loads_layers: Sequence[Sequence[int]], slots: int, fault_threshold: int = 2):
    """Host re-plan of every layer for the live ranks (rebuild_adaptive_plans,
    simulator.py:363-384).  ``R_layers[l]`` is layer l's current replica matrix in
    communicator-rank order and ``node_ids[r]`` the node of communicator rank r
    (ascending).  Returns (new_R_layers, order, transfers, plans) with transfers =
    [((layer, expert), src_node, dst_node)] (plan_state_transfers, migration.py:164-195)."""
    live = list(node_ids)
    if live != sorted(live):
        raise ValueError("communicator ranks must map to ascending node ids")
    spec = ClusterSpec(len(live), slots, min(fault_threshold, len(live)))
    plans = [build_mro_plan(allocate_replicas(list(loads), spec), spec, layer=li)
             for li, loads in enumerate(loads_layers)]
    holdings = {live[r]: {(li, e) for li, R in enumerate(R_layers)
                          for e, row in enumerate(R) if row[r] > 0} for r in range(len(live))}
    cols = [{(li, e) for li, p in enumerate(plans) for e in p.column(c)}
            for c in range(len(live))]
    order = node_order(greedy_node_mapping(holdings, cols, live))
    new_R = [replica_matrix(p, order) for p in plans]
    fetch = {node: cols[c] - holdings[node] for c, node in enumerate(order)}
    owners: dict = {}
    for v in live:
        for item in holdings[v]:
            owners.setdefault(item, []).append(v)
    transfers, _ = plan_state_transfers(fetch, owners)
    return new_R, order, transfers, plans


class Rebalancer:
    """Attach a load window to ``layers`` and re-place their replicas every ``interval``
    steps (call :meth:`step` once per training step; it syncs only when it fires)."""

    def __init__(self, layers: Sequence, slots: int, fault_threshold: int = 2,
                 interval: int = 200):
        self.layers = list(layers)
        self.slots, self.f, self.interval = slots, fault_threshold, interval
        self.since = 0
        self.version = 0
        for layer in self.layers:
            layer.load_window = LoadWindow(layer.E, interval, layer.device)

    def step(self) -> dict | None:
        self.since += 1
        if self.since < self.interval:
            return None
        self.since = 0
        return self.rebalance()

    def rebalance(self) -> dict:
        from .elastic import exchange_expert_state
        loads = [layer.load_window.loads() for layer in self.layers]
        if any(v is None for v in loads):
            return {"event": "rebalance", "detail": "no load recorded", "changed": False}
        first = self.layers[0]
        nodes = list(getattr(first, "node_ids", range(first.world)))
        new_R, order, transfers, _ = plan_rebalance([layer.R for layer in self.layers], nodes,
                                                    loads, self.slots, self.f)
        if all(list(map(list, R)) == [list(r) for r in layer.R]
               for R, layer in zip(new_R, self.layers)):
            return {"event": "rebalance", "detail": "allocation unchanged", "changed": False,
                    "loads": loads}
        if first.world > 1:
            me = nodes[first.rank]
            rank_of = {v: r for r, v in enumerate(nodes)}
            weights = exchange_expert_state(self.layers, transfers, me, rank_of, first.group)
        else:
            weights = [layer.expert_state() for layer in self.layers]
        for layer, R, w in zip(self.layers, new_R, weights):
            layer.set_plan(R, weights=w)
        self.version += 1
        return {"event": "rebalance", "detail": "allocation updated", "changed": True,
                "loads": loads, "order": order, "transfers": len(transfers),
                "bytes": sum(2 * self.layers[li].d * self.layers[li].d_ff * 2 *
                             (1.5 if self.layers[li].activation == "swiglu" else 1)
                             for (li, _), _, _ in transfers)}
