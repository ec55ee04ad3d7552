"""CPU reference arm of the MoE-layer hot path (TEST / BASELINE INFRASTRUCTURE).

Used only by bench.py's ``cpu_baseline`` leg and ``--impl reference``.  It runs the
reference's algorithm end to end on the host cores: integer planning restated in
oracle/dispatch_ref.py (pinned to the reference's golden vectors), then torch-CPU
fp32 gating, per-expert FFN, combine and autograd backward (oracle/moe_ref.py
semantics), exactly the "CPU-baseline plan" of BASELINE.md section 3.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import dispatch_ref as O
from .moe_ref import gate_ref, gelu


def make_weights(E, d, dff, seed=0, std=0.02, bias=None, activation="gelu"):
    g = torch.Generator().manual_seed(seed)
    wg = (torch.randn(E, d, generator=g) * (1.28 / d ** 0.5)).requires_grad_(True)
    bg = (torch.zeros(E) if bias is None else bias.clone().float()).requires_grad_(True)
    w1 = (torch.randn(E, dff, d, generator=g) * std).requires_grad_(True)
    w2 = (torch.randn(E, d, dff, generator=g) * std).requires_grad_(True)
    w3 = (torch.randn(E, dff, d, generator=g) * std).requires_grad_(True) \
        if activation == "swiglu" else None
    return wg, bg, w1, w2, w3


def layer_step(xs, wg, bg, w1, w2, k, R, renorm=False, backward=True, w3=None):
    """One MoE-layer step over N virtual ranks (xs[i] = rank i's tokens): histogram ->
    gather_load_matrix -> compute_dispatch_schedule -> build_shuffle_index -> pack ->
    expert FFN -> combine (-> autograd backward).  Returns total tokens processed."""
    N = len(xs)
    E = wg.shape[0]
    routed, ws, probs = [], [], []
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
    T = O.gather_load_matrix(hist)
    total = 0
    loss = 0.0
    for i, x in enumerate(xs):
        sch = O.compute_dispatch_schedule(i, T, R)
        index = O.build_shuffle_index(sch["D"], routed[i])        # send order
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
        inv = torch.from_numpy(O.invert_permutation(index))
        out = (y[inv].view(x.shape[0], k, -1) * ws[i].unsqueeze(-1)).sum(1)  # combine
        total += x.shape[0]
        loss = loss + (out * out).sum() * 0.5
    if backward:
        loss.backward()
    return total


def run(tokens_per_rank, n_ranks, E, d, dff, k, R, reps=1, seed=0, bias=None, backward=True,
        threads=None, activation="gelu"):
    """Returns (tokens/s, seconds, tokens)."""
    if threads:
        torch.set_num_threads(threads)
    wg, bg, w1, w2, w3 = make_weights(E, d, dff, seed, bias=bias, activation=activation)
    g = torch.Generator().manual_seed(seed + 1)
    xs = [torch.randn(tokens_per_rank, d, generator=g) for _ in range(n_ranks)]
    t0 = time.perf_counter()
    tok = 0
    for _ in range(reps):
        tok += layer_step(xs, wg, bg, w1, w2, k, R, backward=backward, w3=w3)
    dt = time.perf_counter() - t0
    return tok / dt, dt, tok
