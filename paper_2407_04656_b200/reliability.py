"""Recovery probability of a placement under uniformly random node failures
(reference reliability.py).

``recovery_probability_exact`` counts the recoverable failure sets on the GPU
(``lz_recovery_count``: one thread per range of colex-ranked failed-node masks) and
returns the same exact ``Fraction`` as reference reliability.py:68-96, with the same
argument checks and the same ``EnumerationCapError`` contract (the cap is a parameter;
the GPU makes caps of 10^10+ practical).  ``is_recoverable`` and the closed form are
host arithmetic, as in the reference (reliability.py:46-56, 99-125).
"""

from __future__ import annotations

import math
from fractions import Fraction
from typing import Iterable

import torch

from . import _lib
from ._lib import ptr
from .placement import AllocationPlan, ClusterSpec, PlacementPlan

DEFAULT_ENUMERATION_CAP = 10**6   # reliability.py:24


class EnumerationCapError(ValueError):
    """Exact enumeration would exceed the configured subset cap (reliability.py:28-29)."""


def is_recoverable(plan: PlacementPlan, alive_set: Iterable[int]) -> bool:
    """True iff the surviving nodes jointly hold every expert (reliability.py:46-56)."""
    alive = set(alive_set)
    if not alive <= set(range(plan.n_nodes)):
        raise ValueError("alive_set contains unknown node indices")
    covered: set[int] = set()
    for j in alive:
        covered |= plan.col_sets[j]
    return len(covered) == plan.n_experts


def holder_masks(plan: PlacementPlan) -> list[int]:
    """holders[e] = bit mask of the nodes holding expert e."""
    masks = [0] * plan.n_experts
    for j, cs in enumerate(plan.col_sets):
        for e in cs:
            masks[e] |= 1 << j
    return masks


def recovery_probability_exact(plan: PlacementPlan, k_failed: int,
                               enumeration_cap: int = DEFAULT_ENUMERATION_CAP,
                               device=None) -> Fraction:
    """Exact recovery probability under ``k_failed`` uniform node failures
    (reliability.py:68-96), counted on the GPU."""
    n = plan.n_nodes
    if not 0 <= k_failed <= n:
        raise ValueError("k_failed must be in [0, N]")
    total = math.comb(n, n - k_failed)
    if total > enumeration_cap:
        raise EnumerationCapError(
            f"C({n},{n - k_failed}) = {total} exceeds cap {enumeration_cap}; "
            "use recovery_probability_mc")
    if n > 63 or plan.n_experts > 1024:
        raise ValueError("GPU enumeration supports N <= 63 nodes and E <= 1024 experts")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    masks = holder_masks(plan)
    if any(m == 0 for m in masks):
        return Fraction(0, total)      # an expert with no holder is never recoverable
    h = torch.tensor([m if m < 2**63 else m - 2**64 for m in masks], dtype=torch.int64,
                     device=dev)
    good = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.call("lz_recovery_count", ptr(h), len(masks), n, k_failed, ptr(good),
              torch.cuda.current_stream(dev).cuda_stream)
    return Fraction(int(good.item()), total)


def group_sizes(alloc: AllocationPlan, n_nodes: int, slots_per_node: int) -> list[int]:
    """Node-group sizes of the grouped placement (placement.py:89-98)."""
    c = slots_per_node
    n_groups = math.ceil(alloc.n_experts / c)
    srt = alloc.sorted_replicas
    sizes = [srt[i * c] for i in range(n_groups - 1)]
    sizes.append(min(n_nodes - sum(sizes), srt[(n_groups - 1) * c]))
    return sizes


def recovery_probability_closed_form(alloc: AllocationPlan, spec: ClusterSpec,
                                     r_alive: int) -> Fraction:
    """Inclusion-exclusion over missed node groups (reliability.py:99-125)."""
    n = spec.n_nodes
    if not 0 <= r_alive <= n:
        raise ValueError("r_alive must be in [0, N]")
    lengths = group_sizes(alloc, n, spec.slots_per_node)
    denom = math.comb(n, r_alive)
    total = 0
    g = len(lengths)
    for bits in range(1 << g):
        removed = sum(lengths[i] for i in range(g) if bits >> i & 1)
        sign = -1 if bin(bits).count("1") % 2 else 1
        if n - removed >= 0:
            total += sign * math.comb(n - removed, r_alive)
    return Fraction(total, denom)
