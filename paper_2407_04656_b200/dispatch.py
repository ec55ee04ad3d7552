"""Drop-in for ``flexep.dispatch`` (reference: /root/reference/pkg/src/flexep/dispatch.py),
computed by the sm_100a planning kernels of liblz.

The public names, argument meanings, return types and error behaviour follow the
reference module line by line, so reference call sites (``cli.cmd_dispatch``,
``simulator.adaptive_layer_cost``) and reference tests can switch imports:

    ReplicaMatrix              dispatch.py:28-58
    DispatchSchedule           dispatch.py:61-92
    gather_load_matrix         dispatch.py:95-107
    full_dispatch_matrices     dispatch.py:129-159   -> lz_plan_matrices
    compute_dispatch_schedule  dispatch.py:162-196   -> lz_plan_dispatch
    build_shuffle_index        dispatch.py:199-237   -> lz_shuffle_index
    invert_permutation         dispatch.py:240-244   -> lz_invert_permutation
    simulate_all_to_all        dispatch.py:247-283   (host-side consistency check)
    UnroutableTokenError / DispatchConsistencyError  dispatch.py:20-25

Inputs may be nested Python sequences (as in the reference) or torch tensors;
outputs are the reference's immutable types.  The device-resident entry point
used by the MoE layer itself is :func:`plan_device` (no host round trip).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple, Sequence

import torch

from . import _lib

try:  # keep exception identity with the reference when it is importable
    import flexep.dispatch as _ref_dispatch  # type: ignore

    _UnroutableBase = _ref_dispatch.UnroutableTokenError
    _ConsistencyBase = _ref_dispatch.DispatchConsistencyError
except Exception:  # pragma: no cover - reference absent (the GPU box)
    _UnroutableBase = ValueError
    _ConsistencyBase = ValueError


class UnroutableTokenError(_UnroutableBase):
    """Tokens are routed to an expert that has no replica anywhere."""


class DispatchConsistencyError(_ConsistencyBase):
    """Send and receive schedules disagree; indicates corrupted inputs."""


def _check_ragged(rows) -> int:
    width = None
    for row in rows:
        if width is None:
            width = len(row)
        elif len(row) != width:
            raise ValueError("ragged input: rows have differing lengths")
    if width is None:
        raise ValueError("empty input")
    return width


@dataclass(frozen=True)
class ReplicaMatrix:
    """``counts[e][j]``: replicas of expert e hosted on rank j (dispatch.py:28-58)."""

    counts: tuple[tuple[int, ...], ...]

    def __post_init__(self) -> None:
        _check_ragged(self.counts)
        for row in self.counts:
            if any(v < 0 for v in row):
                raise ValueError("replica counts must be non-negative")

    @classmethod
    def from_plan(cls, plan, node_order: Sequence[int] | None = None,
                  ranks: Sequence[int] | None = None) -> "ReplicaMatrix":
        """R from a placement plan (any object with ``n_experts``, ``n_nodes`` and
        ``column(j)``, e.g. ``flexep.placement.PlacementPlan``).

        Without ``node_order`` column j is rank j (the reference, dispatch.py:40-47).
        With ``node_order[col] = node`` (controller.py:447-450) and ``ranks`` (the
        communicator rank of each node, default: position in sorted(node_order)),
        columns are permuted into communicator-rank order -- required because the
        largest-remainder split breaks ties by index (SURVEY.md 8b rank-order trap)."""
        n = plan.n_nodes
        cols = [tuple(plan.column(j)) for j in range(n)]
        if node_order is not None:
            if ranks is None:
                ranks = {node: r for r, node in enumerate(sorted(node_order))}
            else:
                ranks = {node: r for node, r in zip(sorted(node_order), ranks)} \
                    if not isinstance(ranks, dict) else ranks
            perm = [None] * n
            for col, node in enumerate(node_order):
                perm[ranks[node]] = cols[col]
            cols = perm
        rows = tuple(tuple(cols[j].count(e) for j in range(n)) for e in range(plan.n_experts))
        return cls(rows)

    @property
    def n_experts(self) -> int:
        return len(self.counts)

    @property
    def n_ranks(self) -> int:
        return len(self.counts[0])

    def total(self, e: int) -> int:
        return sum(self.counts[e])

    def to_tensor(self, device="cuda") -> torch.Tensor:
        return torch.tensor(self.counts, dtype=torch.int32, device=device)


@dataclass(frozen=True)
class DispatchSchedule:
    """One rank's dispatch decisions (dispatch.py:61-92)."""

    rank: int
    send_counts: tuple[tuple[int, ...], ...]
    send_sizes: tuple[int, ...]
    recv_sizes: tuple[int, ...]
    quota: tuple[int, ...]

    @property
    def n_experts(self) -> int:
        return len(self.send_counts)

    @property
    def n_ranks(self) -> int:
        return len(self.send_sizes)

    def to_dict(self) -> dict:
        return {
            "rank": self.rank,
            "D": [list(row) for row in self.send_counts],
            "s": list(self.send_sizes),
            "recv": list(self.recv_sizes),
            "quota": list(self.quota),
        }


# ---------------------------------------------------------------- helpers


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the Lazarus B200 dispatcher needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _as_i32(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.int32).contiguous()
    return torch.tensor(x, dtype=torch.int32, device=device)


def _tr(t_matrix, replicas) -> tuple[torch.Tensor, torch.Tensor, int, int]:
    """Shape checks of dispatch.py:137-142, then int32 device tensors."""
    dev = _dev()
    counts = replicas.counts if isinstance(replicas, ReplicaMatrix) else replicas
    if isinstance(t_matrix, torch.Tensor):
        E, N = t_matrix.shape
    else:
        E = len(t_matrix)
        N = _check_ragged(t_matrix)
    if isinstance(counts, torch.Tensor):
        Er, Nr = counts.shape
    else:
        Er = len(counts)
        Nr = _check_ragged(counts)
    if E != Er:
        raise ValueError("T and R disagree on expert count")
    if N != Nr:
        raise ValueError("T and R disagree on rank count")
    return _as_i32(t_matrix, dev), _as_i32(counts, dev), E, N


class ExchangeCapacityError(RuntimeError):
    """The plan needs more exchange-buffer rows than are allocated (LZ_ERRF_CAPACITY).
    Every rank sees the same plan and raises together; nothing was exchanged.  Grow the
    buffers to ``rows`` (``MoELayer.reserve``) and re-run the step."""

    def __init__(self, rows: int):
        super().__init__(f"exchange buffers too small: the plan needs {rows} rows")
        self.rows = rows


def _raise_err(flag: int, need: int = 0) -> None:
    if flag & _lib.LZ_ERRF_UNROUTABLE:
        raise UnroutableTokenError("an expert has routed tokens but no replicas")
    if flag & _lib.LZ_ERRF_EXPERT_ID:
        raise ValueError("token routed to unknown expert")
    if flag & _lib.LZ_ERRF_COUNTS:
        raise ValueError("routing list per-expert counts disagree with the schedule")
    if flag & _lib.LZ_ERRF_CAPACITY:
        raise ExchangeCapacityError(need)


def _ws(E: int, N: int, P: int, dev) -> torch.Tensor:
    n = _lib.ctypes.c_size_t(0)
    _lib.call("lz_plan_workspace_bytes", E, N, P, _lib.ctypes.byref(n))
    return torch.empty(int(n.value), dtype=torch.uint8, device=dev)


# ------------------------------------------------------------ device plan


class DevicePlan(NamedTuple):
    """Everything lz_plan_dispatch produces, resident on the device."""

    quota: torch.Tensor        # int64 [E]
    D: torch.Tensor            # int32 [N, E, N]  all senders
    send_sizes: torch.Tensor   # int32 [N]  incl. self
    recv_sizes: torch.Tensor   # int32 [N]  reference convention (self = 0)
    recv_counts: torch.Tensor  # int32 [N]  incl. self
    slot: torch.Tensor         # int32 [P]  send slot of assignment p
    gather: torch.Tensor       # int32 [P]  assignment at send slot s
    dest_row: torch.Tensor     # int32 [P]  row in the destination's expert-major buffer
    dest_rank: torch.Tensor    # int32 [P]  destination rank
    recv_m: torch.Tensor       # int32 [E]
    recv_off: torch.Tensor     # int32 [E+1] padded expert-major offsets (this rank)
    recv_src_off: torch.Tensor  # int32 [E, N]
    recv_stage_off: torch.Tensor  # int32 [E, N]
    recv_cnt: torch.Tensor     # int32 [E, N]
    err: torch.Tensor          # int32 [2]: error bits, rows the exchange needs

    def check(self) -> None:
        """Synchronises; raises the reference's exception on a device error flag."""
        flag, need = self.err.tolist()
        _raise_err(flag, need)

    @property
    def need_rows(self) -> torch.Tensor:
        return self.err[1:]


def plan_device(T: torch.Tensor, R: torch.Tensor, rank: int, routed: torch.Tensor | None,
                align: int = 128, stream=None, cap_rows: int = 0) -> DevicePlan:
    """Asynchronous full plan for ``rank`` on the current stream (no host sync).
    T, R: int32 [E, N] device tensors in communicator-rank order; routed: int32 [P].
    cap_rows > 0: rows of the exchange buffers (overflow -> ExchangeCapacityError at
    :meth:`DevicePlan.check`, identically on every rank)."""
    E, N = T.shape
    dev = T.device
    P = 0 if routed is None else routed.numel()
    i32 = dict(dtype=torch.int32, device=dev)
    quota = torch.empty(E, dtype=torch.int64, device=dev)
    D = torch.empty((N, E, N), **i32)
    send_sizes, recv_sizes, recv_counts = (torch.empty(N, **i32) for _ in range(3))
    slot = torch.empty(P, **i32)
    gather = torch.empty(P, **i32)
    dest_row = torch.empty(P, **i32)
    dest_rank = torch.empty(P, **i32)
    recv_m = torch.empty(E, **i32)
    recv_off = torch.empty(E + 1, **i32)
    recv_src_off, recv_stage_off, recv_cnt = (torch.empty((E, N), **i32) for _ in range(3))
    err = torch.zeros(2, **i32)
    ws = _ws(E, N, P, dev)
    _lib.call("lz_plan_dispatch", _lib.ptr(T), _lib.ptr(R), E, N, rank,
              _lib.ptr(routed) if P else None, P, align, int(cap_rows), err[1:].data_ptr(),
              _lib.ptr(quota), _lib.ptr(D),
              _lib.ptr(send_sizes), _lib.ptr(recv_sizes), _lib.ptr(recv_counts),
              _lib.ptr(slot) if P else None, _lib.ptr(gather) if P else None,
              _lib.ptr(dest_row) if P else None, _lib.ptr(dest_rank) if P else None,
              _lib.ptr(recv_m), _lib.ptr(recv_off),
              _lib.ptr(recv_src_off), _lib.ptr(recv_stage_off), _lib.ptr(recv_cnt),
              _lib.ptr(err), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream))
    return DevicePlan(quota, D, send_sizes, recv_sizes, recv_counts, slot, gather, dest_row,
                      dest_rank, recv_m, recv_off, recv_src_off, recv_stage_off, recv_cnt, err)


# ------------------------------------------------------- reference API


def gather_load_matrix(per_rank_counts: Sequence[Sequence[int]]) -> tuple[tuple[int, ...], ...]:
    """T[e][j] from per-rank E-vectors (dispatch.py:95-107).  The multi-GPU layer
    does this with one NCCL all-gather of the on-device histograms (comm.py)."""
    _check_ragged(per_rank_counts)
    n_ranks = len(per_rank_counts)
    n_experts = len(per_rank_counts[0])
    return tuple(tuple(int(per_rank_counts[j][e]) for j in range(n_ranks))
                 for e in range(n_experts))


def full_dispatch_matrices(t_matrix, replicas) -> list[list[list[int]]]:
    """result[i][e][j]: tokens of e from i to j, for all senders (dispatch.py:129-159)."""
    T, R, E, N = _tr(t_matrix, replicas)
    quota = torch.empty(E, dtype=torch.int64, device=T.device)
    D = torch.empty((N, E, N), dtype=torch.int32, device=T.device)
    err = torch.zeros(1, dtype=torch.int32, device=T.device)
    _lib.call("lz_plan_matrices", _lib.ptr(T), _lib.ptr(R), E, N, _lib.ptr(quota), _lib.ptr(D),
              _lib.ptr(err), _lib.stream_ptr())
    _raise_err(int(err.item()))
    return D.tolist()


def compute_dispatch_schedule(rank: int, t_matrix, replicas) -> DispatchSchedule:
    """Rank ``rank``'s schedule from the shared (T, R) (dispatch.py:162-196)."""
    T, R, E, N = _tr(t_matrix, replicas)
    plan = plan_device(T, R, 0, None) if not 0 <= rank < N else plan_device(T, R, rank, None)
    plan.check()  # raises UnroutableTokenError first, as the reference does
    if not 0 <= rank < N:
        raise ValueError("rank out of range")
    D = plan.D[rank].tolist()
    return DispatchSchedule(
        rank=rank,
        send_counts=tuple(tuple(r) for r in D),
        send_sizes=tuple(plan.send_sizes.tolist()),
        recv_sizes=tuple(plan.recv_sizes.tolist()),
        quota=tuple(plan.quota.tolist()),
    )


def build_shuffle_index(schedule: DispatchSchedule, routed_experts) -> list[int]:
    """Gather indices turning local order into send order (dispatch.py:199-237)."""
    dev = _dev()
    E, N = schedule.n_experts, schedule.n_ranks
    expected = sum(sum(r) for r in schedule.send_counts)
    routed = _as_i32(routed_experts, dev).reshape(-1)
    P = routed.numel()
    if P != expected:
        raise ValueError(f"routing list has {P} tokens, schedule covers {expected}")
    D = _as_i32(schedule.send_counts, dev)
    slot = torch.empty(P, dtype=torch.int32, device=dev)
    gather = torch.empty(P, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = _ws(E, N, P, dev)
    _lib.call("lz_shuffle_index", _lib.ptr(D), E, N, _lib.ptr(routed) if P else None, P,
              _lib.ptr(slot) if P else None, _lib.ptr(gather) if P else None, _lib.ptr(err),
              _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    flag = int(err.item())
    if flag & _lib.LZ_ERRF_EXPERT_ID:
        raise ValueError("token routed to unknown expert")
    if flag & _lib.LZ_ERRF_COUNTS:
        raise ValueError("routing list per-expert counts disagree with the schedule")
    return gather.tolist()


def invert_permutation(index) -> list[int]:
    """dispatch.py:240-244, on the device."""
    dev = _dev()
    idx = _as_i32(index, dev).reshape(-1)
    out = torch.empty_like(idx)
    _lib.call("lz_invert_permutation", _lib.ptr(idx), idx.numel(), _lib.ptr(out),
              _lib.stream_ptr())
    return out.tolist()


def simulate_all_to_all(schedules: Sequence[DispatchSchedule]) -> list[list[list[int]]]:
    """Cross-check all ranks' schedules; returns received[j][e][i] (dispatch.py:247-283).
    Pure host bookkeeping over already-computed schedules (the reference's test
    harness of the all-to-all); the real exchange is NCCL in comm.py."""
    n_ranks = len(schedules)
    if n_ranks == 0:
        return []
    n_experts = schedules[0].n_experts
    for s in schedules:
        if s.n_ranks != n_ranks or s.n_experts != n_experts:
            raise DispatchConsistencyError("schedules have mismatched shapes")
    for i, si in enumerate(schedules):
        for j in range(n_ranks):
            if i != j and si.send_sizes[j] != schedules[j].recv_sizes[i]:
                raise DispatchConsistencyError(
                    f"rank {i} sends {si.send_sizes[j]} tokens to rank {j}, "
                    f"rank {j} expects {schedules[j].recv_sizes[i]}")
    return [[[schedules[i].send_counts[e][j] for i in range(n_ranks)] for e in range(n_experts)]
            for j in range(n_ranks)]


__all__ = [
    "DevicePlan", "DispatchConsistencyError", "ExchangeCapacityError", "DispatchSchedule", "ReplicaMatrix",
    "UnroutableTokenError", "build_shuffle_index", "compute_dispatch_schedule",
    "full_dispatch_matrices", "gather_load_matrix", "invert_permutation", "plan_device",
    "simulate_all_to_all",
]
