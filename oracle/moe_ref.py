"""torch-CPU fp32 restatement of the float stages of the MoE layer (TEST INFRASTRUCTURE).

No reference code exists for these stages; they follow
PAPER.md:94-99 (top-k gate, weighted combine), :143 (replicas share one weight copy),
:296 (expert-gradient all-reduce over the replica group) and GPT-2's tanh GELU MLP.
Parity for them is "restated", with tolerances written in each test.
"""

from __future__ import annotations

import numpy as np
import torch


def gate_ref(logits: torch.Tensor, k: int, renorm: bool = False):
    """softmax over E, top-k chosen on the fp32 logits, ties -> lower expert id."""
    lg = logits.detach().float().cpu()
    Tn, E = lg.shape
    # stable sort on -logit keeps the lower id first among equal logits
    order = np.argsort(-lg.numpy(), axis=1, kind="stable")[:, :k]
    idx = torch.from_numpy(order.astype(np.int64))
    probs = torch.softmax(lg, dim=1)
    w = torch.gather(probs, 1, idx)
    if renorm:
        w = w / w.sum(dim=1, keepdim=True)
    return idx.to(torch.int32), w, probs


def gelu(x: torch.Tensor) -> torch.Tensor:
    return torch.nn.functional.gelu(x, approximate="tanh")


def ffn_ref(x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor, w3=None) -> torch.Tensor:
    """One expert: gelu(x W1^T) W2^T (GPT) or (silu(x W1^T) * x W3^T) W2^T (Mixtral);
    W1, W3 [d_ff, d], W2 [d, d_ff] (fp32)."""
    if w3 is None:
        return gelu(x @ w1.t()) @ w2.t()
    return (torch.nn.functional.silu(x @ w1.t()) * (x @ w3.t())) @ w2.t()


def moe_forward_ref(x, wg, bg, w1, w2, k: int, renorm: bool = False, idx=None, w3=None):
    """Full layer in fp32 on the CPU.  x [T, d]; wg [E, d]; bg [E]; w1 [E, d_ff, d];
    w2 [E, d, d_ff].  Returns (out, idx, w, probs).  Differentiable w.r.t. all inputs
    (the top-k selection is treated as constant, as in the GPU backward).  If ``idx``
    is given the routing is forced (used when bf16 logits near-ties could flip)."""
    logits = x @ wg.t() + (bg if bg is not None else 0.0)
    probs = torch.softmax(logits, dim=1)
    if idx is None:
        idx, _, _ = gate_ref(logits, k, renorm)
    idx = idx.long()
    w = torch.gather(probs, 1, idx)
    if renorm:
        w = w / w.sum(dim=1, keepdim=True)
    out = torch.zeros_like(x)
    for e in range(w1.shape[0]):
        tok, slot = (idx == e).nonzero(as_tuple=True)
        if tok.numel() == 0:
            continue
        y = ffn_ref(x[tok], w1[e], w2[e], None if w3 is None else w3[e])
        out = out.index_add(0, tok, y * w[tok, slot].unsqueeze(1))
    return out, idx.to(torch.int32), w, probs
