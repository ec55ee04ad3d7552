"""N EP ranks on ONE GPU, in lockstep, through the product's own per-rank step
(SURVEY.md 4.4 "single-GPU multi-rank loopback").

``MoELayer``'s forward and backward are generators that yield a request wherever ranks
interact (layer.py).  ``LoopbackWorld`` advances N of them -- one ``MoELayer`` per
virtual rank, each with its own plan column, hosted experts and exchange buffers -- one
request at a time and serves the requests on the single device:

    HIST       the all-gather: T = stack of the N histograms
    SYMM       every rank's exchange buffers carved out of one allocation; the peer
               tables hold the other ranks' real device addresses, so the fused P2P
               dispatch, the arrival flags, the scattering GEMM epilogues and the
               combine-backward stores are the multi-GPU kernels writing "remote" rows
    SYNC       nothing: lockstep already orders every rank's launches before the next
               phase (e.g. all dispatches + arrival signals before any arrival GEMM)
    BARRIER    each rank's ``lz_peer_barrier`` kernel on its own stream, released after
               every rank's earlier work (signal + wait through the real flags)
    EXPERT_AR  the replica-group gradient sum over each expert's owner set (fp32)
    ALLREDUCE  sum over ranks (router gradients)
    A2A        row all-to-all-v by device copies (the ``LZ_EXCHANGE=nccl`` regroup path)

so the default N > 1 path (and the NCCL-exchange variant) runs forward AND backward on
one B200 at any N (2 ... 8) and is compared with the oracle on the gathered batch
(tests/test_loopback_gpu.py).  A rank can be "lost" mid-step (``lose``): the survivors'
device waits time out through the watchdog control block, the step is discarded
(``StepAbortedError``), and ``shrink`` re-plans over the survivors (elastic.py recipe)
and moves the expert state, as after a real failure.
"""

from __future__ import annotations

import torch

from . import _lib, comm
from .comm import A2A, ALLREDUCE, BARRIER, EXPERT_AR, HIST, SYMM, SYNC, WAIT
from .layer import MoELayer, _backward_steps, _forward_steps


class PeerLostError(RuntimeError):
    """A collective was requested while a rank is lost (the NCCL-timeout analogue)."""


class LoopbackBuffers(comm.SymmetricRows):
    """Rank r's view of the world's exchange buffers: the SymmetricRows interface over
    slices of one device allocation (no IPC: every "peer" address is on this GPU)."""

    def __init__(self, world: "LoopbackWorld", r: int):   # noqa: D401 -- no super().__init__
        a = world._alloc
        n = world.n
        self.rows, self.d, self.nbuf = a["rows"], a["d"], a["nbuf"]
        self.n, self.rank = n, r
        self.t = a["t"][r]
        self.host_ptrs = a["host_ptrs"]
        self.ptrs = a["ptrs"]
        self.ret = a["ret"][r]
        self.ret_ptrs = a["ret_ptrs"]
        self.flags = a["flags"][r]
        self.flag_peers = a["flag_peers"]
        self.epoch = a["epoch"][r]
        self.bar_count = a["bar"][r]


class LoopbackRank:
    """Fabric handle of virtual rank r (what ``MoELayer(fabric=...)`` takes)."""

    group = None

    def __init__(self, world: "LoopbackWorld", r: int):
        self.loop, self.rank, self.world = world, r, world.n

    def replica_groups(self, R, max_ctas=None):
        return None   # the world sums over owner sets itself (EXPERT_AR)

    def run(self, gen):
        raise RuntimeError("loopback ranks advance in lockstep: use LoopbackWorld.step/run")


class LoopbackWorld:
    def __init__(self, n: int, device=None):
        self.n = n
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.ranks = [LoopbackRank(self, r) for r in range(n)]
        self.streams = [torch.cuda.Stream(device=self.device)]   # the barrier stream
        self._alloc = None
        self.lost: set[int] = set()
        self.requests = 0

    def fabric(self, r: int) -> LoopbackRank:
        return self.ranks[r]

    # ------------------------------------------------------------ layers
    def make_layers(self, d_model, d_ff, n_experts, top_k, replicas, **kw) -> list[MoELayer]:
        """One MoELayer per virtual rank (same seed: identical router and expert copies)."""
        return [MoELayer(d_model, d_ff, n_experts, top_k, replicas=replicas,
                         fabric=self.fabric(r), device=self.device, **kw)
                for r in range(self.n)]

    @torch.no_grad()
    def step(self, layers, xs, douts=None, lose: dict | None = None):
        """Forward (and backward when ``douts`` is given) of every rank in lockstep.
        Returns outs, or (outs, grads) with grads[r] = (dx, dwg, dbg, dW1, dW2) -- the
        expert grads already summed over each expert's owner set, the router grads over
        all ranks.  ``lose = {rank: n}``: that rank is lost after issuing n requests of
        the forward (e.g. after its dispatch, before the combine)."""
        sts = [{} for _ in layers]
        outs = self.run([_forward_steps(L, x, L.wg, L.bg, L.w1, L.w2, st)
                         for L, x, st in zip(layers, xs, sts)], lose)
        if douts is None:
            return outs
        grads = self.run([_backward_steps(L, st, x.contiguous(), L.wg, L.w1, L.w2, g)
                          for L, st, x, g in zip(layers, sts, xs, douts)])
        return outs, grads

    def run(self, gens, lose: dict | None = None) -> list:
        """Advance the generators one request at a time, all ranks together."""
        n = len(gens)
        results = [None] * n
        done = [False] * n
        res = [None] * n
        issued = [0] * n
        while not all(done):
            reqs = {}
            for r in range(n):
                if done[r]:
                    continue
                if lose and r in lose and issued[r] >= lose[r]:
                    gens[r].close()
                    done[r] = True
                    self.lost.add(r)
                    continue
                try:
                    reqs[r] = gens[r].send(res[r])
                    issued[r] += 1
                except StopIteration as stop:
                    results[r] = stop.value
                    done[r] = True
            if not reqs:
                break
            kinds = {q[0] for q in reqs.values()}
            if len(kinds) != 1:
                raise RuntimeError(f"virtual ranks diverged: {sorted(kinds)}")
            self.requests += 1
            out = self.serve(kinds.pop(), reqs)
            for r in reqs:
                res[r] = out.get(r)
        return results

    # ------------------------------------------------------------ requests
    def serve(self, kind: str, reqs: dict) -> dict:
        if kind in (HIST, SYMM, EXPERT_AR, ALLREDUCE, A2A) and self.lost:
            raise PeerLostError(f"{kind} with lost ranks {sorted(self.lost)}")
        ranks = sorted(reqs)
        if kind == HIST:
            T = torch.stack([reqs[r][1] for r in ranks], dim=1).contiguous()
            return {r: T for r in ranks}
        if kind == SYNC:
            return {}
        if kind == BARRIER:
            # the live ranks' barriers as ONE launch (a warp per rank, lz_peer_barrier_
            # colocated): ranks that wait on each other are never separate launches on one
            # GPU.  It starts after every rank's earlier work (all request streams) and
            # every request stream continues after it.
            a = self._alloc
            tab = torch.tensor([ranks,
                                [a["bar"][r].data_ptr() for r in ranks],
                                [a["flags"][r][2].data_ptr() for r in ranks]],
                               dtype=torch.int64, device=self.device)
            rk = tab[0].to(torch.int32)
            waits = list({id(reqs[r][2]): reqs[r][2] for r in ranks}.values())
            st0 = self.streams[0]
            st0.wait_stream(torch.cuda.current_stream(self.device))
            for st in waits:
                st0.wait_stream(st)
            with torch.cuda.stream(st0):
                _lib.call("lz_peer_barrier_colocated", _lib.ptr(a["flag_peers"][2]), self.n,
                          _lib.ptr(rk), len(ranks), _lib.ptr(tab[1]), _lib.ptr(tab[2]),
                          st0.cuda_stream)
                tab.record_stream(st0)
                rk.record_stream(st0)
            for st in waits:
                st.wait_stream(st0)
            return {}
        if kind == SYMM:
            rows = max(reqs[r][1] for r in ranks)
            _, _, nbuf, d, dev = reqs[ranks[0]]
            self._allocate(rows, nbuf, d, dev)
            return {r: LoopbackBuffers(self, r) for r in ranks}
        if kind == EXPERT_AR:
            layers = {r: reqs[r][1] for r in ranks}
            grads = {r: reqs[r][2] for r in ranks}
            E = layers[ranks[0]].E
            lo, hi = reqs[ranks[0]][3] if len(reqs[ranks[0]]) > 3 else (0, E)
            for gi in range(len(grads[ranks[0]])):
                for e in range(lo, hi):
                    owners = [(r, layers[r].local_ids.index(e)) for r in ranks
                              if e in layers[r].local_ids]
                    if len(owners) < 2:
                        continue
                    acc = sum(grads[r][gi][p].float() for r, p in owners)
                    for r, p in owners:
                        grads[r][gi][p].copy_(acc)
            return {r: [] for r in ranks}
        if kind == WAIT:
            return {}
        if kind == ALLREDUCE:
            acc = sum(reqs[r][1].float() for r in ranks)
            for r in ranks:
                reqs[r][1].copy_(acc)
            return {}
        if kind == A2A:
            # rank r: out <- rows from every j (out_splits[j] of them), inp -> every j
            def offsets(splits):
                o, acc = [], 0
                for v in splits:
                    o.append(acc)
                    acc += int(v)
                return o
            ooff = {r: offsets(reqs[r][3]) for r in ranks}
            ioff = {r: offsets(reqs[r][4]) for r in ranks}
            for r in ranks:
                out, _, out_splits, _ = reqs[r][1:]
                for j in ranks:
                    cnt = int(out_splits[j])
                    if cnt:
                        src = reqs[j][2][ioff[j][r]:ioff[j][r] + cnt]
                        out[ooff[r][j]:ooff[r][j] + cnt].copy_(src)
            return {r: reqs[r][1] for r in ranks}
        raise ValueError(f"unknown exchange request {kind!r}")

    def _allocate(self, rows: int, nbuf: int, d: int, device) -> None:
        n = self.n
        self._alloc = None
        t = torch.empty((n, nbuf, rows, d), dtype=torch.bfloat16, device=device)
        stride = rows * d * 2
        base = [t[r].data_ptr() for r in range(n)]
        host_ptrs = [[b + i * stride for b in base] for i in range(nbuf)]
        ret = torch.empty((n, rows), dtype=torch.int64, device=device)
        flags = torch.zeros((n, 3, n), dtype=torch.int32, device=device)
        fb = [flags[r].data_ptr() for r in range(n)]
        self._alloc = {
            "rows": rows, "nbuf": nbuf, "d": d, "t": t, "host_ptrs": host_ptrs,
            "ptrs": torch.tensor(host_ptrs, dtype=torch.int64, device=device),
            "ret": ret,
            "ret_ptrs": torch.tensor([ret[r].data_ptr() for r in range(n)], dtype=torch.int64,
                                     device=device),
            "flags": flags,
            "flag_peers": torch.tensor([[b + i * n * 4 for b in fb] for i in range(3)],
                                       dtype=torch.int64, device=device),
            "epoch": torch.zeros((n, 1), dtype=torch.int32, device=device),
            "bar": torch.zeros((n, 1), dtype=torch.int32, device=device),
        }

    # ------------------------------------------------------------ elastic
    def shrink(self, layers, loads, slots: int, fault_threshold: int = 2, optimizers=None):
        """Survivors of the lost ranks form a new world; the host re-plans with the
        reference recipe (elastic.replan) and every newly hosted expert's weights -- and,
        with ``optimizers`` (one per rank), its optimizer state -- are copied from a
        surviving owner (the NCCL send/recv of elastic.exchange_expert_state, here device
        copies); optimizers are re-pointed at the new parameters (elastic.remap_optimizer).
        Returns (new_world, survivor layers, report)."""
        from .elastic import expert_slices, optimizer_state_keys, remap_optimizer, replan, \
            transfer_schedule
        survivors = [r for r in range(self.n) if r not in self.lost]
        holdings = {r: {e for e, row in enumerate(layers[r].R) if row[r] > 0}
                    for r in survivors}
        plan, order, R = replan(loads, survivors, holdings, slots, fault_threshold)
        transfers, orphans = transfer_schedule(R, survivors, holdings)
        world = LoopbackWorld(len(survivors), self.device)
        opts = optimizers or [None] * self.n
        keys = optimizer_state_keys(layers[survivors[0]], opts[survivors[0]])
        kept = {r: expert_slices(layers[r], opts[r], keys) for r in survivors}
        new_layers = []
        for nr, r in enumerate(survivors):
            L = layers[r]
            slices = dict(kept[r])
            for e, src, dst in transfers:
                if dst == r:
                    slices[e] = [t.clone() for t in kept[src][e]]
            L.set_fabric(world.fabric(nr))
            L.node_ids = survivors
            info = L.set_plan(R, weights={e: (v[0], v[1]) for e, v in slices.items()})
            if opts[r] is not None:
                remap_optimizer(opts[r], L, info, slices, keys)
            new_layers.append(L)
        report = {"live": survivors, "order": order, "transfers": len(transfers),
                  "checkpoint_fallback": orphans, "replicas": list(plan.replica_counts)}
        return world, new_layers, report
