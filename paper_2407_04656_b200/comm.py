"""Collective plumbing of the multi-GPU MoE layer (torch.distributed over NCCL).

    load all-gather    gather_load_matrix (dispatch.py:95-107) as one all-gather of
                       the E-int histograms K1 produces
    a2a-v              the padding-free flexible all-to-all (SPEC.md:372-380,
                       simulate_all_to_all dispatch.py:247-283 is its reference check)
    replica-group AR   expert gradients summed over the expert's owner ranks
                       {j : R[e][j] > 0}, one sub-communicator per
                       distinct owner set, cached per plan version

All functions work on any backend torch.distributed supports (NCCL on the B200
box, gloo in the CPU tests of the host logic).
"""

from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist


def world(group=None) -> tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def allgather_hist(hist: torch.Tensor, group=None) -> torch.Tensor:
    """Per-rank expert histograms (int32 [E]) -> load matrix T [E, N] (int32)."""
    rank, n = world(group)
    if n == 1:
        return hist.view(-1, 1).contiguous()
    out = torch.empty(n * hist.numel(), dtype=hist.dtype, device=hist.device)
    dist.all_gather_into_tensor(out, hist.contiguous(), group=group)
    return out.view(n, -1).t().contiguous()


def all_to_all_rows(out: torch.Tensor, inp: torch.Tensor, out_splits: Sequence[int],
                    in_splits: Sequence[int], group=None) -> torch.Tensor:
    """Row all-to-all-v: rank i sends in_splits[j] rows to rank j and receives
    out_splits[j] rows from rank j (no padding)."""
    dist.all_to_all_single(out, inp, [int(v) for v in out_splits], [int(v) for v in in_splits],
                           group=group)
    return out


class SymmetricRows:
    """``nbuf`` row buffers [rows, d] (bf16) allocated in NVLink-mapped symmetric memory
    (torch symmetric memory: cuMem + IPC handles, one mapping per peer).  ``peers(b)``
    is a device int64 [N] array of every rank's address of buffer b, consumed by the
    fused P2P dispatch/combine kernels; ``barrier()`` is a device-side cross-rank
    barrier on the current stream (orders P2P writes before the peers read; bounded by
    the watchdog control block, ``_lib.control``).

    Collective: every rank must construct it with the same ``rows`` (``ProcessFabric``
    agrees on the maximum first)."""

    def __init__(self, group, nbuf: int, rows: int, d: int, device):
        import torch.distributed._symmetric_memory as symm
        try:
            symm.enable_symm_mem_for_group(group.group_name)
        except Exception:
            pass
        self.rows, self.d, self.nbuf = rows, d, nbuf
        self.t = symm.empty((nbuf, rows, d), dtype=torch.bfloat16, device=device)
        self.h = symm.rendezvous(self.t, group)
        n = self.h.world_size
        base = [self.h.get_remote_tensor(r, (nbuf, rows, d), torch.bfloat16).data_ptr()
                for r in range(n)]
        stride = rows * d * 2
        self.host_ptrs = [[b + i * stride for b in base] for i in range(nbuf)]
        self.ptrs = torch.tensor(self.host_ptrs, dtype=torch.int64, device=device)
        # return map (int64 per receive row: source rank << 32 | source assignment), written
        # by the senders' dispatch, read by the owner's scattering GEMM epilogue
        self.ret = symm.empty((rows,), dtype=torch.int64, device=device)
        self.hr = symm.rendezvous(self.ret, group)
        self.ret_ptrs = torch.tensor(
            [self.hr.get_remote_tensor(r, (rows,), torch.int64).data_ptr() for r in range(n)],
            dtype=torch.int64, device=device)
        # flags [3 (dispatch arrivals, combine-backward arrivals, barrier), n senders], this
        # rank's step epoch and barrier count
        self.n = n
        self.rank = self.h.rank
        self.flags = symm.empty((3, n), dtype=torch.int32, device=device)
        self.flags.zero_()
        self.hf = symm.rendezvous(self.flags, group)
        fb = [self.hf.get_remote_tensor(r, (3, n), torch.int32).data_ptr() for r in range(n)]
        self.flag_peers = torch.tensor([[b + i * n * 4 for b in fb] for i in range(3)],
                                       dtype=torch.int64, device=device)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)
        self.bar_count = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        self.hf.barrier(channel=0)   # every rank's flags are zero before anyone signals

    def buf(self, i: int) -> torch.Tensor:
        return self.t[i]

    def peers(self, i: int) -> torch.Tensor:
        return self.ptrs[i]

    def peers_host(self, i: int) -> list[int]:
        return self.host_ptrs[i]

    def barrier(self, stream=None) -> None:
        from . import ops
        ops.peer_barrier(self.flag_peers[2], self.n, self.rank, self.bar_count, self.flags[2],
                         stream)


def owner_sets(R: Sequence[Sequence[int]]) -> list[tuple[int, ...]]:
    """owners[e] = ranks hosting at least one replica of expert e."""
    return [tuple(j for j, v in enumerate(row) if v > 0) for row in R]


_PG_CACHE: dict = {}


class ReplicaGroups:
    """Sub-communicators for the replica-group gradient all-reduce.

    Built collectively (every rank creates every group, in the same sorted order,
    as torch.distributed requires) once per plan; experts sharing an owner set share
    a communicator and their gradients travel in one bucket."""

    def __init__(self, R: Sequence[Sequence[int]], group=None, backend: str | None = None,
                 max_ctas: int | None = None):
        """max_ctas (NCCL): cap on the CTAs each all-reduce may occupy -- the backward GEMMs
        that overlap the all-reduces leave exactly that many SMs free, so the persistent
        GEMM CTAs and NCCL's never queue behind each other."""
        self.rank, self.n = world(group)
        self.owners = owner_sets(R)
        self.sets = sorted({o for o in self.owners if len(o) > 1})
        self.groups: dict[tuple[int, ...], object] = {}
        if self.n > 1:
            base = dist.get_process_group_ranks(group) if group is not None else list(range(self.n))
            opts = None
            if max_ctas and (backend or dist.get_backend(group)) == "nccl":
                opts = dist.ProcessGroupNCCL.Options()
                opts.config.max_ctas = int(max_ctas)
                opts.config.min_ctas = 1
                opts.is_high_priority_stream = True
            parent = getattr(group, "group_name", "default") if group is not None else "default"
            for s in self.sets:
                # communicators are cached per (parent group, member set): a re-plan that
                # keeps an owner set reuses its communicator instead of leaking a new one
                key = (parent, tuple(base[j] for j in s), backend, max_ctas)
                pg = _PG_CACHE.get(key)
                if pg is None:
                    pg = dist.new_group([base[j] for j in s], backend=backend, pg_options=opts)
                    _PG_CACHE[key] = pg
                if self.rank in s:
                    self.groups[s] = pg

    def buckets(self, local_ids: Sequence[int]) -> list[tuple[object, list[int]]]:
        """[(process group, local expert positions)] for this rank."""
        out: dict[tuple[int, ...], list[int]] = {}
        for pos, e in enumerate(local_ids):
            s = self.owners[e]
            if len(s) > 1:
                out.setdefault(s, []).append(pos)
        return [(self.groups[s], pos) for s, pos in sorted(out.items())]

    def allreduce(self, grads: Sequence[torch.Tensor], local_ids: Sequence[int]) -> None:
        """Sum each local expert's gradient slices ([E_loc, ...] tensors) over the
        expert's owner ranks, in place."""
        for w in self.allreduce_async(grads, local_ids):
            w.wait()

    def allreduce_async(self, grads: Sequence[torch.Tensor], local_ids: Sequence[int],
                        id_range: tuple[int, int] | None = None) -> list:
        """As :meth:`allreduce`, issued asynchronously (NCCL streams); returns the works
        whose ``wait()`` makes the current stream wait for the sums.  ``id_range`` = (lo, hi):
        only experts lo <= e < hi (the same id range on every rank, so every owner set's
        members issue the same sequence)."""
        works: list = []
        if self.n == 1:
            return works
        for pg, pos in self.buckets(local_ids):
            if id_range is not None:
                pos = [q for q in pos if id_range[0] <= local_ids[q] < id_range[1]]
                if not pos:
                    continue
            # runs of consecutive EXPERT IDS: every member rank hosts all of them, so they
            # are contiguous local positions on every member and all members issue the same
            # sequence of equally sized in-place all-reduces (no copies)
            ids = [local_ids[p] for p in pos]
            runs, a = [], 0
            for i in range(1, len(ids) + 1):
                if i == len(ids) or ids[i] != ids[i - 1] + 1:
                    runs.append((pos[a], pos[i - 1] + 1))
                    a = i
            for g in grads:
                for a, b in runs:
                    works.append(dist.all_reduce(g[a:b], group=pg, async_op=True))
        return works


# ---------------------------------------------------------------- exchange fabric

# Requests a rank's layer step yields wherever ranks interact (layer._forward_steps /
# _backward_steps).  A fabric serves them: ProcessFabric for one process per GPU
# (NCCL + NVLink symmetric memory), loopback.LoopbackWorld for N ranks on one GPU.
HIST = "hist"            # (hist [E] int32)                 -> T [E, N]
SYNC = "sync"            # ()  every rank's launches so far precede what follows
BARRIER = "barrier"      # (sym, stream)  device barrier over the exchange buffers
SYMM = "symm"            # (rows, nbuf, d)                  -> exchange buffers
EXPERT_AR = "expert_ar"  # (layer, grads[, (lo, hi) expert ids])  replica-group sum -> works
WAIT = "wait"            # (works)
ALLREDUCE = "allreduce"  # (flat tensor)  in-place sum over all ranks
A2A = "a2a"              # (out, inp, out_splits, in_splits)  row all-to-all-v


class ProcessFabric:
    """One rank per process (the product path): serves the layer's requests with
    torch.distributed (NCCL) collectives and the NVLink symmetric-memory buffers."""

    def __init__(self, group=None):
        self.group = group
        self.rank, self.world = world(group)

    def replica_groups(self, R, max_ctas=None):
        return ReplicaGroups(R, self.group, max_ctas=max_ctas) if self.world > 1 else None

    def run(self, gen):
        """Drive one rank's step generator to completion; returns its value."""
        res = None
        while True:
            try:
                req = gen.send(res)
            except StopIteration as stop:
                return stop.value
            res = self.serve(req)

    def serve(self, req):
        kind = req[0]
        if kind == HIST:
            return allgather_hist(req[1], self.group)
        if kind == SYNC:
            return None
        if kind == BARRIER:
            req[1].barrier(req[2])
            return None
        if kind == SYMM:
            rows, nbuf, d, device = req[1:]
            t = torch.tensor([rows], dtype=torch.int64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)   # ranks agree
            return SymmetricRows(self.group, nbuf, int(t.item()), d, device)
        if kind == EXPERT_AR:
            layer, grads = req[1], req[2]
            ids = req[3] if len(req) > 3 else None
            return layer.replica_groups.allreduce_async(grads, layer.local_ids, ids)
        if kind == WAIT:
            for w in req[1]:
                w.wait()
            return None
        if kind == ALLREDUCE:
            dist.all_reduce(req[1], group=self.group)
            return None
        if kind == A2A:
            return all_to_all_rows(*req[1:], group=self.group)
        raise ValueError(f"unknown exchange request {kind!r}")
