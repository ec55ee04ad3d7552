"""Integer oracle: restatement of the reference dispatcher (TEST INFRASTRUCTURE).

Every function cites the reference lines it restates (paths relative to
``/root/reference/pkg/src/flexep``).  Results are returned as plain Python
ints / nested lists or int64 numpy arrays so they compare exactly against the
golden vectors in ``tests/golden/dispatch_golden.json`` (produced by running
the reference itself, see ``tests/golden/make_golden.py``).

Conventions kept from the reference:
  * ``T[e][j]``  tokens routed to expert e that originate on rank j
  * ``R[e][j]``  replicas of expert e hosted on rank j
  * ``D[i][e][j]`` tokens of expert e sent from rank i to rank j
  * ``recv_sizes[rank] == 0`` (dispatch.py:181-184)
"""

from __future__ import annotations

from math import ceil
from typing import Sequence

import numpy as np


class UnroutableTokenError(ValueError):
    """dispatch.py:20-21"""


class DispatchConsistencyError(ValueError):
    """dispatch.py:24-25"""


def _width(rows) -> int:
    """core.py:358-368 (check_ragged)."""
    width = None
    for row in rows:
        if width is None:
            width = len(row)
        elif len(row) != width:
            raise ValueError("ragged input: rows have differing lengths")
    if width is None:
        raise ValueError("empty input")
    return width


def split_proportionally(total: int, weights: Sequence[int]) -> list[int]:
    """Largest-remainder split; ties to the lower index.  core.py:321-341."""
    if total < 0:
        raise ValueError("total must be non-negative")
    if any(w < 0 for w in weights):
        raise ValueError("weights must be non-negative")
    wsum = sum(weights)
    if wsum == 0:
        if total == 0:
            return [0] * len(weights)
        raise ValueError("cannot split a positive total over all-zero weights")
    base = [total * w // wsum for w in weights]
    rem = [total * w - b * wsum for w, b in zip(weights, base)]
    left = total - sum(base)
    # rank each index by (remainder desc, index asc); the first `left` get +1
    for i in range(len(weights)):
        ahead = sum(1 for j in range(len(weights))
                    if rem[j] > rem[i] or (rem[j] == rem[i] and j < i))
        if ahead < left:
            base[i] += 1
    return base


def quotas(T: Sequence[Sequence[int]], R: Sequence[Sequence[int]]) -> list[int]:
    """q_e = ceil(t_e / r_e) (float division as in the reference), 0 when r_e == 0;
    UnroutableTokenError when t_e > 0 and r_e == 0.  dispatch.py:143-151."""
    out = []
    for e in range(len(T)):
        t_e, r_e = sum(T[e]), sum(R[e])
        if t_e > 0 and r_e == 0:
            raise UnroutableTokenError(f"expert {e} has {t_e} routed tokens but no replicas")
        out.append(ceil(t_e / r_e) if r_e else 0)
    return out


def dispatch_row(i: int, t_row, r_row, q: int) -> list[int]:
    """Sender i, one expert: keep min(T, q*R) locally, split the overflow over the
    other ranks by residual capacity.  dispatch.py:110-126."""
    n = len(t_row)
    cap = [q * r_row[j] for j in range(n)]
    keep = min(t_row[i], cap[i])
    over = t_row[i] - keep
    row = [0] * n
    row[i] = keep
    if over:
        resid = [cap[j] - min(cap[j], t_row[j]) if j != i else 0 for j in range(n)]
        for j, v in enumerate(split_proportionally(over, resid)):
            row[j] += v
    return row


def full_dispatch_matrices(T, R) -> list[list[list[int]]]:
    """D[i][e][j] for every sender i.  dispatch.py:129-159."""
    E = len(T)
    if E != len(R):
        raise ValueError("T and R disagree on expert count")
    N = _width(T)
    if N != _width(R):
        raise ValueError("T and R disagree on rank count")
    q = quotas(T, R)
    return [[dispatch_row(i, T[e], R[e], q[e]) for e in range(E)] for i in range(N)]


def compute_dispatch_schedule(rank: int, T, R) -> dict:
    """One rank's schedule in the reference's ``to_dict`` form
    {rank, D, s, recv, quota}.  dispatch.py:162-196 and :85-92."""
    D = full_dispatch_matrices(T, R)
    E, N = len(T), len(R[0])
    if not 0 <= rank < N:
        raise ValueError("rank out of range")
    mine = D[rank]
    s = [sum(mine[e][j] for e in range(E)) for j in range(N)]
    recv = [sum(D[j][e][rank] for e in range(E)) if j != rank else 0 for j in range(N)]
    return {"rank": rank, "D": [list(r) for r in mine], "s": s, "recv": recv,
            "quota": quotas(T, R)}


def build_shuffle_index(send_counts, routed) -> np.ndarray:
    """index[slot] = local assignment position; destination-major, expert-major,
    original order within a group.  dispatch.py:199-237 (including its
    validation errors)."""
    D = np.asarray(send_counts, dtype=np.int64)
    E, N = D.shape
    routed = np.asarray(routed, dtype=np.int64).reshape(-1)
    expected = D.sum(axis=1)
    if routed.size != int(expected.sum()):
        raise ValueError(f"routing list has {routed.size} tokens, schedule covers {int(expected.sum())}")
    if routed.size and (routed.min() < 0 or routed.max() >= E):
        raise ValueError("token routed to unknown expert")
    counts = np.bincount(routed, minlength=E)
    if not np.array_equal(counts, expected):
        raise ValueError("routing list per-expert counts disagree with the schedule")
    order = np.argsort(routed, kind="stable")          # positions grouped by expert
    first = np.concatenate([[0], np.cumsum(counts)[:-1]])
    taken = np.zeros(E, dtype=np.int64)
    parts = []
    for j in range(N):
        for e in range(E):
            c = int(D[e, j])
            if c:
                parts.append(order[first[e] + taken[e]: first[e] + taken[e] + c])
                taken[e] += c
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def invert_permutation(index) -> np.ndarray:
    """dispatch.py:240-244."""
    index = np.asarray(index, dtype=np.int64)
    out = np.empty_like(index)
    out[index] = np.arange(index.size, dtype=np.int64)
    return out


def gather_load_matrix(per_rank_counts) -> tuple:
    """T[e][j] from per-rank E-vectors.  dispatch.py:95-107."""
    _width(per_rank_counts)
    N, E = len(per_rank_counts), len(per_rank_counts[0])
    return tuple(tuple(int(per_rank_counts[j][e]) for j in range(N)) for e in range(E))


def simulate_all_to_all(schedules) -> list:
    """received[j][e][i]; raises on send/recv disagreement.  dispatch.py:247-283.
    ``schedules`` are dicts as returned by :func:`compute_dispatch_schedule`."""
    N = len(schedules)
    if N == 0:
        return []
    E = len(schedules[0]["D"])
    for s in schedules:
        if len(s["s"]) != N or len(s["D"]) != E:
            raise DispatchConsistencyError("schedules have mismatched shapes")
    for i, si in enumerate(schedules):
        for j in range(N):
            if i != j and si["s"][j] != schedules[j]["recv"][i]:
                raise DispatchConsistencyError(
                    f"rank {i} sends {si['s'][j]} tokens to rank {j}, "
                    f"rank {j} expects {schedules[j]['recv'][i]}")
    return [[[schedules[i]["D"][e][j] for i in range(N)] for e in range(E)] for j in range(N)]


def send_slots(send_counts, routed) -> np.ndarray:
    """slot[p] = position of local assignment p in the send buffer
    (= invert_permutation(build_shuffle_index(...)))."""
    return invert_permutation(build_shuffle_index(send_counts, routed))


def recv_layout(D_all, rank: int, align: int = 1):
    """Receive side of the flexible all-to-all on ``rank`` in the layout the GPU
    path uses for the expert GEMMs: expert-major, source-major inside an expert,
    each expert segment padded to ``align`` rows.  Returns (m_e, pad_off[E+1],
    src_off[E][N]) -- counts only; the reference stops at counts (a9)."""
    D = np.asarray(D_all, dtype=np.int64)        # [N, E, N]
    N, E, _ = D.shape
    m = D[:, :, rank].sum(axis=0)                # tokens of e received on rank
    padded = (m + align - 1) // align * align
    pad_off = np.concatenate([[0], np.cumsum(padded)])
    src_off = np.zeros((E, N), dtype=np.int64)
    for e in range(E):
        src_off[e] = pad_off[e] + np.concatenate([[0], np.cumsum(D[:, e, rank])[:-1]])
    return m, pad_off, src_off


def adaptive_layer_cost(R, layer_tokens: Sequence[int], n_ranks: int) -> tuple[int, int]:
    """(max per-node compute tokens, cross-node tokens) of one layer under the flexible
    dispatch, tokens split uniformly over the ranks.  simulator.py:198-219 (R is
    ReplicaMatrix.from_plan(plan).counts, dispatch.py:40-47)."""
    T = [split_proportionally(int(t), [1] * n_ranks) for t in layer_tokens]
    D = full_dispatch_matrices(T, R)
    node = [0] * n_ranks
    cross = 0
    for i in range(n_ranks):
        for row in D[i]:
            for j in range(n_ranks):
                node[j] += row[j]
                if j != i:
                    cross += row[j]
    return max(node), cross


def step_time_adaptive(Rs: dict, layer_loads: dict, n_ranks: int, alpha: float, beta: float,
                       overhead: float) -> float:
    """step_time_model(strategy="adaptive") (simulator.py:248-266): overhead +
    sum over layers (sorted) of alpha * max_node + beta * cross."""
    total = overhead
    for layer, tokens in sorted(layer_loads.items()):
        max_node, cross = adaptive_layer_cost(Rs[layer], tokens, n_ranks)
        total += alpha * max_node + beta * cross
    return total
