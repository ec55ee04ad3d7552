"""CPU reference arm of the MoE-layer hot path (TEST / BASELINE INFRASTRUCTURE).

Used only by bench.py's ``cpu_baseline`` leg and ``--impl reference``.  It runs the
reference's algorithm end to end on the host cores:

  * integer stages -- replica allocation + MRO placement (allocation.py:75-107,
    placement.py:101-138), gather_load_matrix, compute_dispatch_schedule,
    build_shuffle_index, invert_permutation (dispatch.py:95-244) -- through the
    UNMODIFIED reference package ``flexep`` from ``baseline/_ref``
    (tools/install_reference.sh) when it is present (``kind = "reference"``), else
    through the restatement in oracle/dispatch_ref.py pinned to the reference's golden
    vectors (``kind = "port"``);
  * float stages -- torch-CPU fp32 gating, per-expert FFN, combine and autograd backward
    (oracle/moe_ref.py semantics; the reference has no float code), the "CPU-baseline
    plan" of BASELINE.md section 3.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np
import torch

from . import dispatch_ref as O
from .moe_ref import gate_ref, gelu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def reference_flexep():
    """The unmodified reference package from baseline/_ref, or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "flexep")) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import flexep.allocation
        import flexep.core
        import flexep.dispatch
        import flexep.placement
        if "baseline" not in flexep.__file__:
            return None
        return flexep
    except Exception:
        return None


class _Planner:
    """The integer stages, either flexep (reference) or the oracle port."""

    def __init__(self, impl: str = "auto"):
        self.fx = reference_flexep() if impl in ("auto", "reference") else None
        if impl == "reference" and self.fx is None:
            raise RuntimeError("flexep not found in baseline/_ref (tools/install_reference.sh)")
        self.kind = "reference" if self.fx is not None else "port"

    def replicas(self, loads, n_ranks, slots, f):
        if self.fx is not None:
            fx = self.fx
            spec = fx.core.ClusterSpec(n_ranks, slots, min(f, n_ranks))
            plan = fx.placement.build_mro_plan(fx.allocation.allocate_replicas(list(loads), spec),
                                               spec)
            return fx.dispatch.ReplicaMatrix.from_plan(plan)
        from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
        return replica_matrix(plan_for_loads(list(loads), n_ranks, slots, f))

    def gather(self, hist):
        return (self.fx.dispatch.gather_load_matrix(hist) if self.fx is not None
                else O.gather_load_matrix(hist))

    def send_index(self, rank, T, R, routed):
        """(index: send slot -> local assignment, inverse) for one rank."""
        if self.fx is not None:
            d = self.fx.dispatch
            sch = d.compute_dispatch_schedule(rank, T, R)
            index = d.build_shuffle_index(sch, routed.tolist())
            return np.asarray(index, dtype=np.int64), np.asarray(d.invert_permutation(index))
        sch = O.compute_dispatch_schedule(rank, T, R)
        index = O.build_shuffle_index(sch["D"], routed)
        return index, O.invert_permutation(index)


def make_weights(E, d, dff, seed=0, std=0.02, bias=None, activation="gelu"):
    g = torch.Generator().manual_seed(seed)
    wg = (torch.randn(E, d, generator=g) * (1.28 / d ** 0.5)).requires_grad_(True)
    bg = (torch.zeros(E) if bias is None else bias.clone().float()).requires_grad_(True)
    w1 = (torch.randn(E, dff, d, generator=g) * std).requires_grad_(True)
    w2 = (torch.randn(E, d, dff, generator=g) * std).requires_grad_(True)
    w3 = (torch.randn(E, dff, d, generator=g) * std).requires_grad_(True) \
        if activation == "swiglu" else None
    return wg, bg, w1, w2, w3


def layer_step(xs, wg, bg, w1, w2, k, R, renorm=False, backward=True, w3=None, planner=None):
    """One MoE-layer step over N ranks (xs[i] = rank i's tokens): histogram ->
    gather_load_matrix -> compute_dispatch_schedule -> build_shuffle_index -> pack ->
    expert FFN -> combine (-> autograd backward).  Returns total tokens processed."""
    planner = planner or _Planner("port")
    E = wg.shape[0]
    routed, ws = [], []
    for x in xs:
        logits = x @ wg.t() + bg
        idx, _, _ = gate_ref(logits.detach(), k, renorm)
        p = torch.softmax(logits, 1)
        w = torch.gather(p, 1, idx.long())
        if renorm:
            w = w / w.sum(1, keepdim=True)
        routed.append(idx.reshape(-1).numpy())
        ws.append(w)
    hist = [np.bincount(r, minlength=E).tolist() for r in routed]
    T = planner.gather(hist)
    total = 0
    loss = 0.0
    for i, x in enumerate(xs):
        index, inv = planner.send_index(i, T, R, routed[i])      # send order, its inverse
        tok = torch.from_numpy(index // k)
        send = x[tok]                                             # pack
        exp_of = torch.from_numpy(routed[i][index])
        y = torch.empty_like(send)
        for e in range(E):                                        # expert FFN (any replica)
            sel = (exp_of == e).nonzero(as_tuple=True)[0]
            if sel.numel():
                if w3 is None:
                    h = gelu(send[sel] @ w1[e].t())
                else:
                    h = torch.nn.functional.silu(send[sel] @ w1[e].t()) * (send[sel] @ w3[e].t())
                y = y.index_copy(0, sel, h @ w2[e].t())
        out = (y[torch.from_numpy(inv)].view(x.shape[0], k, -1) * ws[i].unsqueeze(-1)).sum(1)
        total += x.shape[0]
        loss = loss + (out * out).sum() * 0.5
    if backward:
        loss.backward()
    return total


def run(tokens_per_rank, n_ranks, E, d, dff, k, loads, slots, f=2, reps=1, seed=0, bias=None,
        backward=True, threads=None, activation="gelu", impl="auto"):
    """Returns (tokens/s, seconds, tokens, kind).  The replica plan (from ``loads``) is
    built with the same planner as the dispatch and is inside the timed region."""
    if threads:
        torch.set_num_threads(threads)
    planner = _Planner(impl)
    wg, bg, w1, w2, w3 = make_weights(E, d, dff, seed, bias=bias, activation=activation)
    g = torch.Generator().manual_seed(seed + 1)
    xs = [torch.randn(tokens_per_rank, d, generator=g) for _ in range(n_ranks)]
    t0 = time.perf_counter()
    tok = 0
    for _ in range(reps):
        R = planner.replicas(loads, n_ranks, slots, f)
        tok += layer_step(xs, wg, bg, w1, w2, k, R, backward=backward, w3=w3, planner=planner)
    dt = time.perf_counter() - t0
    return tok / dt, dt, tok, planner.kind


def slots_for(cfg, n_ranks) -> int:
    return math.ceil(cfg["slot_factor"] * cfg["E"] / n_ranks)
