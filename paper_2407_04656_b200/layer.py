"""MoELayer: the Lazarus MoE-layer hot path on B200 (fwd + bwd + replica-group sync).

Per rank, per step:
    K1 router_gate      x . wg^T + b -> softmax / top-k -> idx, w, probs, hist
    all-gather hist     -> T [E, N]                                   (N > 1)
    K2 plan_device      bit-exact reference dispatch: D, sizes, slot, dest_row
    K3 pack             rows -> expert-major padded receive buffer (N = 1 directly;
                        N > 1 straight into the owners' NVLink buffers, or send buffer ->
                        NCCL a2a-v -> segment regroup)
    K4 grouped GEMM x2  X W1^T (+GELU/SwiGLU epilogue, keeps the backward factor), A W2^T
                        (N > 1: its epilogue stores each row back on its source rank)
    K7 combine          weighted sum of the k outputs
backward:
    K8 combine_bwd -> K5 dgrad (dY W2 . act'(H), dH W1) + K6 wgrad (variable-K, per
    expert) -> K8 dispatch/gate bwd -> router wgrad -> replica-group all-reduce of the
    expert grads, DP all-reduce of the router grads.

One weight copy per (expert, rank) hosting it: R[e][rank] > 1 only
raises the capacity the planner gives that rank.

The per-rank step is written ONCE, as two generators (``_forward_steps`` /
``_backward_steps``) that yield a request (``comm.HIST``, ``SYNC``, ``BARRIER``, ...)
wherever ranks interact.  A fabric serves the requests: ``comm.ProcessFabric`` (one
process per GPU: NCCL + NVLink symmetric memory -- the product path) or
``loopback.LoopbackWorld`` (N ranks on one GPU in lockstep, same kernels, same flags and
device barriers) -- so the multi-rank path is verifiable on a single B200.

Failure semantics: every cross-rank wait on the device is bounded by the
watchdog control block (``_lib.control``); a lost peer makes the step's waits time out,
``check()`` raises ``StepAbortedError`` and the caller discards the step, shrinks and
re-plans (``elastic``).  Exchange buffers are sized from the balanced share of the
assignments (``LZ_CAPACITY_SLACK``); a plan that needs more rows is detected on the
device identically on every rank (``ExchangeCapacityError`` at ``check()``), nothing is
exchanged, and ``reserve()`` grows the buffers for the re-run.
"""

from __future__ import annotations

import math
import os

import torch

from . import _lib, comm, ops
from .comm import A2A, ALLREDUCE, BARRIER, EXPERT_AR, HIST, SYMM, SYNC, WAIT
from .dispatch import DevicePlan, ReplicaMatrix, plan_device

ALIGN = ops.ALIGN


class StepAbortedError(RuntimeError):
    """A cross-rank wait of this step timed out or was aborted (a peer was lost mid-step,
    PAPER.md:297).  The step's results are garbage: discard it, shrink and re-plan."""

    def __init__(self, status: dict):
        super().__init__(f"step aborted: {status}")
        self.status = status


def _expert_weights(seed: int, e: int, shape, std: float, device) -> torch.Tensor:
    """Deterministic per-expert init: every owner rank of expert e builds the same copy."""
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + e)
    return (torch.randn(shape, generator=g, device=device) * std).to(torch.bfloat16)


def interleave_swiglu(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """W1 (gate), W3 (up) [..., F, K] -> [..., 2F, K], alternating 128-row blocks, so one
    256-wide GEMM N tile carries gate and up of the same 128 hidden units."""
    F, K = w1.shape[-2:]
    lead = w1.shape[:-2]
    return torch.stack([w1.reshape(*lead, F // 128, 128, K), w3.reshape(*lead, F // 128, 128, K)],
                       dim=-3).reshape(*lead, 2 * F, K)


def deinterleave_swiglu(w13: torch.Tensor):
    F2, K = w13.shape[-2:]
    lead = w13.shape[:-2]
    v = w13.reshape(*lead, F2 // 256, 2, 128, K)
    return v[..., 0, :, :].reshape(*lead, F2 // 2, K), v[..., 1, :, :].reshape(*lead, F2 // 2, K)


def init_expert(seed: int, e: int, d: int, d_ff: int, std: float, device, activation: str):
    """Deterministic expert e weights (identical on every owner rank)."""
    if activation == "gelu":
        return (_expert_weights(seed, 2 * e, (d_ff, d), std, device),
                _expert_weights(seed, 2 * e + 1, (d, d_ff), std, device))
    w1 = _expert_weights(seed, 3 * e, (d_ff, d), std, device)
    w3 = _expert_weights(seed, 3 * e + 1, (d_ff, d), std, device)
    return interleave_swiglu(w1, w3), _expert_weights(seed, 3 * e + 2, (d, d_ff), std, device)


class MoELayer(torch.nn.Module):
    def __init__(self, d_model: int, d_ff: int, n_experts: int, top_k: int = 2, *,
                 replicas=None, group=None, renorm: bool = False, seed: int = 0,
                 init_std: float = 0.02, router_bias=None, device=None, exchange: str | None = None,
                 activation: str = "gelu", router_std: float | None = None, fabric=None):
        super().__init__()
        if activation not in ("gelu", "swiglu"):
            raise ValueError("activation must be 'gelu' (GPT MLP) or 'swiglu' (Mixtral)")
        self.activation = activation
        if d_model % 256 or d_ff % 256:
            raise ValueError("d_model and d_ff must be multiples of 256 (GEMM tile)")
        if not 1 <= top_k <= min(n_experts, _lib.LZ_MAX_TOPK) or n_experts > 64:
            raise ValueError("need 1 <= top_k <= min(E, 8) and E <= 64")
        self.d, self.d_ff, self.E, self.k = d_model, d_ff, n_experts, top_k
        self.renorm = renorm
        self.seed = seed
        self.init_std = init_std
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.device = dev
        self.set_fabric(fabric if fabric is not None else comm.ProcessFabric(group))
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.wg = torch.nn.Parameter(
            (torch.randn(n_experts, d_model, generator=g, device=dev) *
             (init_std if router_std is None else router_std)).bfloat16())
        bias = torch.zeros(n_experts, device=dev) if router_bias is None else \
            torch.as_tensor(router_bias, dtype=torch.float32, device=dev)
        self.bg = torch.nn.Parameter(bias.float().clone())
        self.w1 = None
        self.w2 = None
        self.last_plan: DevicePlan | None = None
        self.exchange = exchange or os.environ.get("LZ_EXCHANGE", "p2p")
        self._fwd_version = 0
        self.stage_events: list | None = None
        self.load_window = None   # rebalance.LoadWindow, attached by rebalance.Rebalancer
        # P2P exchange: return expert outputs from the GEMM epilogues (default) instead of
        # reading them back over NVLink in the combine / dispatch backward
        self.scatter = os.environ.get("LZ_P2P_SCATTER", "1") != "0"
        # SMs the backward GEMMs leave to NCCL while the expert-gradient all-reduce runs
        self.overlap_reserve = int(os.environ.get("LZ_OVERLAP_SMS", "16"))
        # dX GEMM first, then the dispatch backward + router weight gradient on a side
        # stream while the two weight-gradient GEMMs run (they fill the GEMM tails; cfg2
        # graph replay 6.12 -> 6.04 ms/step at N = 1, tools/tail_ab.py)
        self.tail_overlap = os.environ.get("LZ_TAIL_OVERLAP", "1") != "0"
        # N > 1: the same reordering (dX GEMM second, dispatch backward + router weight
        # gradient on the side stream) -- the last expert-gradient all-reduce is then no
        # longer hidden behind the dX GEMM.  Same-box A/B (tools/step_ab.py): N = 4
        # 7.79 -> 7.30 ms/step, N = 2 7.09 -> 7.18 (cfg3 37.0 -> 38.0), so "auto" = N >= 4;
        # LZ_TAIL_OVERLAP_NX=1 / 0 forces it on / off (None = auto, decided per step from the
        # live world size, so it follows an elastic shrink)
        nx = os.environ.get("LZ_TAIL_OVERLAP_NX", "auto")
        self.tail_overlap_nx = None if nx == "auto" else nx == "1"
        # without the tail overlap (N > 1 default), LZ_EARLY_RWGRAD=1: the gate backward right
        # after the combine backward (lz_gate_bwd) and the router weight gradient on a side
        # stream from there (it needs only dlogits and x).  Bit-identical gradients; same-box
        # A/B at N = 2 (tools/step_ab.py): 7.07 vs 7.16 and 7.10 vs 7.06 ms/step -- within
        # noise (the side kernel only gets SMs in the persistent GEMMs' tails), so off
        self.early_router_wgrad = os.environ.get("LZ_EARLY_RWGRAD", "0") == "1"
        # with the tail overlap at N > 1, LZ_SPLIT_WGRAD=1: the last weight-gradient GEMM as two
        # launches split by expert id, so half of its all-reduce overlaps the other half's
        # GEMM.  Bit-identical; same-box A/B at N = 4 7.43 -> 7.38 ms/step (within noise): off
        self.split_last_wgrad = os.environ.get("LZ_SPLIT_WGRAD", "0") == "1"
        self._tail_stream = None
        # exchange buffers: rows = slack x this rank's assignments (+ expert padding); the
        # planner detects a larger need on the device and reserve() grows them
        self.capacity_slack = float(os.environ.get("LZ_CAPACITY_SLACK", "1.25"))
        self._rows_wanted: int | None = None
        self.set_plan(replicas)

    # ------------------------------------------------------------- fabric / plan
    def set_fabric(self, fabric) -> None:
        """Attach the exchange fabric (a new communicator after an elastic shrink): the
        exchange buffers of the old one are dropped."""
        self.fabric = fabric
        self.group = getattr(fabric, "group", None)
        self.rank, self.world = fabric.rank, fabric.world
        self._symm = None
        if self.world > 1 and self.device.type == "cuda":
            _lib.control()   # bounded cross-rank waits record their failures here

    def set_plan(self, replicas, weights: dict | None = None) -> dict:
        """Install a (new) replica matrix in communicator-rank order.  Experts this rank
        keeps retain their weights; newly hosted experts take ``weights[e] = (w1, w2)``
        (state migrated from a surviving owner) or the deterministic init.  No kernel is
        recompiled: E and N are runtime arguments of every kernel.

        ``w1``/``w2`` become NEW Parameters (their leading dimension is the number of
        hosted experts).  Returns ``{"params": [w1, w2], "replaced": [old w1, old w2],
        "local_ids": [...]}`` so a caller can rebuild its optimizer param groups
        (``elastic.remap_optimizer`` moves the per-expert optimizer state)."""
        if replicas is None:
            R = [[1] * self.world for _ in range(self.E)]
        elif isinstance(replicas, ReplicaMatrix):
            R = [list(r) for r in replicas.counts]
        else:
            R = [list(r) for r in replicas]
        if len(R) != self.E or any(len(r) != self.world for r in R):
            raise ValueError(f"replica matrix must be {self.E} x {self.world}")
        for e, row in enumerate(R):
            if sum(row) == 0:
                raise ValueError(f"expert {e} has no replica")
        old = {}
        replaced = [self.w1, self.w2]
        old_ids = list(getattr(self, "local_ids", []))
        if self.w1 is not None:
            for pos, e in enumerate(self.local_ids):
                old[e] = (self.w1.data[pos], self.w2.data[pos])
        self.R = R
        self.R_dev = torch.tensor(R, dtype=torch.int32, device=self.device)
        self.local_ids = [e for e in range(self.E) if R[e][self.rank] > 0]
        ext = self.local_ids + [self.E]
        self._off_index = torch.tensor(ext, dtype=torch.long, device=self.device)
        self._all_local = len(self.local_ids) == self.E   # off = recv_off (no gather launch)
        w1s, w2s = [], []
        for e in self.local_ids:
            if weights is not None and e in weights:
                a, b = weights[e]
            elif e in old:
                a, b = old[e]
            else:
                a, b = init_expert(self.seed, e, self.d, self.d_ff, self.init_std, self.device,
                                   self.activation)
            w1s.append(a)
            w2s.append(b)
        # gelu:   w1[g] = W1_e [d_ff, d];  swiglu: w1[g] = W1_e|W3_e interleaved in 128-row
        # blocks [2 d_ff, d];  w2[g] = W2_e [d, d_ff] (row-major, K contiguous for fwd)
        self.w1 = torch.nn.Parameter(torch.stack(w1s).contiguous())
        self.w2 = torch.nn.Parameter(torch.stack(w2s).contiguous())
        # LZ_NCCL_MAX_CTAS caps the CTAs of the replica-group all-reduces (0: NCCL default);
        # 32 measured best next to the GEMMs that leave LZ_OVERLAP_SMS SMs free (cfg3, N=2)
        max_ctas = int(os.environ.get("LZ_NCCL_MAX_CTAS", "32")) or None
        self.replica_groups = self.fabric.replica_groups(R, max_ctas=max_ctas)
        return {"params": [self.w1, self.w2], "replaced": replaced,
                "local_ids": list(self.local_ids), "old_local_ids": old_ids}

    def exchange_mode(self) -> str:
        """'local' (N = 1), 'p2p' (fused NVLink dispatch/combine through symmetric memory,
        the default for N > 1) or 'nccl' (send buffer + NCCL all-to-all-v + regroup)."""
        if self.world == 1:
            return "local"
        return self.exchange

    def exchange_rows(self, Tn: int) -> int:
        """Rows of every exchange buffer: slack x the balanced share of the assignments
        (each rank receives N.Tn.k / N on average) + one GEMM tile of padding per expert.
        Fixed at first use (agreed over ranks) until ``reserve`` grows it."""
        if self._rows_wanted is None:
            self._rows_wanted = _capacity(math.ceil(self.capacity_slack * Tn * self.k) +
                                          self.E * (ALIGN - 1))
        return self._rows_wanted

    def reserve(self, rows: int) -> None:
        """Grow the exchange buffers to ``rows`` (ExchangeCapacityError.rows) -- called
        by every rank after the same error; the next forward reallocates collectively."""
        self._rows_wanted = max(self._rows_wanted or 0, _capacity(int(rows * 1.05) + ALIGN))

    def expert_state(self) -> dict:
        return {e: (self.w1.data[p], self.w2.data[p]) for p, e in enumerate(self.local_ids)}

    def check(self) -> None:
        """Raise if the last step failed (syncs): a lost peer / abort (StepAbortedError)
        first, then the reference's exceptions and ExchangeCapacityError from the plan."""
        if self.world > 1:
            st = _lib.control_status()
            if st["timeout"] or st["aborted"] or st["watchdog"]:
                raise StepAbortedError(st)
        if self.last_plan is not None:
            self.last_plan.check()

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return _MoEFunction.apply(x, self.wg, self.bg, self.w1, self.w2, self)

    # ------------------------------------------------------------- stats
    def layer_cost(self) -> tuple[int, int]:
        """(max node tokens, cross-node tokens) of the last plan on its real routing --
        the two terms of the reference's time model (simulator.py:198-219, cost.py)."""
        from .cost import plan_cost
        mx, cross = plan_cost(self.last_plan.D)
        return int(mx), int(cross)

    def imbalance(self) -> float:
        """max_j recv_j / mean_j recv_j of the last plan."""
        p = self.last_plan
        if p is None:
            return float("nan")
        recv = p.D.sum(dim=(0, 1)).float()
        return float(recv.max() / recv.mean().clamp_min(1))


def lzh_num_sms() -> int:
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


_NVTX = os.environ.get("LZ_NVTX", "0") == "1"   # NVTX ranges / marks for nsys & ncu


def _mark(layer, name: str, stream=None) -> None:
    """Stage timing (bench --breakdown): CUDA event on ``stream`` (default: current); with
    LZ_NVTX=1 also an NVTX mark named after the stage that just ended."""
    if _NVTX:
        torch.cuda.nvtx.mark(f"lz.{name}")
    if layer.stage_events is not None:
        s = stream if stream is not None else torch.cuda.current_stream()
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        layer.stage_events.append((name, e, s.cuda_stream))


def stage_breakdown(events) -> dict:
    """{stage: ms}: a stage is the time since the previous mark ON THE SAME STREAM (the
    side-stream stages of the backward tail are timed on the side stream)."""
    out: dict = {}
    last: dict = {}
    for name, ev, sid in events:
        prev = last.get(sid)
        last[sid] = ev
        if prev is None or name in ("fwd_start", "bwd_start", "side_start"):
            continue
        out[name] = out.get(name, 0.0) + prev.elapsed_time(ev)
    return out


def _capacity(rows: int) -> int:
    return (rows + ALIGN - 1) // ALIGN * ALIGN


def _forward_steps(layer: MoELayer, x, wg, bg, w1, w2, st: dict):
    """One rank's forward; yields exchange requests (comm.*) and returns the output.
    Everything the backward needs goes into ``st``."""
    if not x.is_cuda or x.dtype != torch.bfloat16 or x.dim() != 2:
        raise ValueError("x must be a CUDA bf16 [tokens, d_model] tensor")
    x = x.contiguous()
    Tn, d = x.shape
    k, E, G = layer.k, layer.E, len(layer.local_ids)
    N, rank = layer.world, layer.rank
    mode = layer.exchange_mode()
    dev = x.device
    _mark(layer, "fwd_start")
    idx, w, probs, hist = ops.router_gate(x, wg, bg, k, layer.renorm)
    _mark(layer, "gate")
    T = yield (HIST, hist)
    if layer.load_window is not None:   # routing history for the periodic rebalance
        layer.load_window.record(T)
    _mark(layer, "hist_allgather")
    sym = None
    if mode == "p2p":
        rows = layer.exchange_rows(Tn)
        if layer._symm is None or layer._symm.rows < rows:
            layer._symm = None
            layer._symm = yield (SYMM, rows, 4, d, dev)
        sym = layer._symm
    plan = plan_device(T, layer.R_dev, rank, idx.view(-1), ops.row_align(),
                       cap_rows=sym.rows if sym is not None else 0)
    layer.last_plan = plan
    off = plan.recv_off.contiguous() if layer._all_local else \
        plan.recv_off.index_select(0, layer._off_index).contiguous()
    _mark(layer, "plan")
    P = Tn * k
    sizes = None
    self_rows = None
    scatter = mode == "p2p" and layer.scatter
    if mode == "local":
        cap = _capacity(P + E * (ALIGN - 1))
        X = torch.empty((cap, d), dtype=torch.bfloat16, device=dev)
        Y = torch.empty((cap, d), dtype=torch.bfloat16, device=dev)
        ops.pack(x, plan.dest_row, k, X, plan.recv_m, plan.recv_off)
    elif mode == "p2p":
        # fused dispatch: rows go straight into the destination's symmetric buffer, and
        # the owner learns where each row came from (return map for the scatter GEMMs)
        layer._fwd_version += 1
        cap = sym.rows
        X, Y = sym.buf(0), sym.buf(1)
        if scatter:
            # no barrier: each sender publishes an arrival flag after its dispatch and
            # the first GEMM runs the tiles of our own rows while the rest arrive
            ops.epoch_bump(sym.epoch)
            ops.pack_p2p_ret(x, plan.dest_rank, plan.dest_row, k, sym.peers(0), X,
                             plan.recv_m, plan.recv_off, sym.ret_ptrs, sym.ret, rank,
                             plan.slot)
            ops.signal_peers(sym.flag_peers[0], N, rank, sym.epoch)
            self_rows = torch.stack([plan.recv_src_off[:, rank],
                                     plan.recv_src_off[:, rank] + plan.recv_cnt[:, rank]],
                                    1).index_select(0, layer._off_index[:-1]).contiguous()
            yield (SYNC,)
        else:
            ops.pack_p2p(x, plan.dest_rank, plan.dest_row, k, sym.peers(0), X, plan.recv_m,
                         plan.recv_off)
            yield (BARRIER, sym, torch.cuda.current_stream(dev))
    else:
        # NCCL exchange: one D2H of the counts (+ error flags) per layer forward
        host = torch.cat([plan.send_sizes, plan.recv_counts, plan.err,
                          plan.recv_cnt.max().view(1)]).cpu()
        if int(host[2 * N]):
            plan.check()
        send_sizes = host[:N].tolist()
        recv_counts = host[N:2 * N].tolist()
        max_seg = int(host[2 * N + 2])
        sizes = (send_sizes, recv_counts, max_seg)
        n_recv = sum(recv_counts)
        cap = _capacity(n_recv + E * (ALIGN - 1))
        send = torch.empty((P, d), dtype=torch.bfloat16, device=dev)
        ops.pack(x, plan.slot, k, send)
        stage = torch.empty((n_recv, d), dtype=torch.bfloat16, device=dev)
        yield (A2A, stage, send, recv_counts, send_sizes)
        X = torch.empty((cap, d), dtype=torch.bfloat16, device=dev)
        Y = torch.empty((cap, d), dtype=torch.bfloat16, device=dev)
        ops.zero_pad_rows(X, plan.recv_m, plan.recv_off)
        ops.copy_segments(stage, X, plan.recv_stage_off, plan.recv_src_off, plan.recv_cnt,
                          max_seg)
        del send, stage
    _mark(layer, "dispatch")
    d_ff = layer.d_ff
    swi = layer.activation == "swiglu"
    H = torch.empty((cap, 2 * d_ff if swi else d_ff), dtype=torch.bfloat16, device=dev)
    A = torch.empty((cap, d_ff), dtype=torch.bfloat16, device=dev)
    if G > 0:
        epi1 = _lib.LZ_EPI_SWIGLU if swi else _lib.LZ_EPI_GELU
        if scatter:
            ops.grouped_gemm_arrival(X, w1, off, A, self_rows, sym.flags[0], sym.epoch,
                                     aux=H, epilogue=epi1)
            # GEMM + combine all-to-all in one kernel: the epilogue stores every output
            # row into its source rank's return buffer (row = source assignment)
            ops.grouped_gemm_scatter(A, w2, off, Y, sym.ret, sym.peers(1), sym.peers_host(1),
                                     sym.rows)
        else:
            ops.grouped_gemm_rows(X, w1, off, A, aux=H, epilogue=epi1)
            ops.grouped_gemm_rows(A, w2, off, Y)
    _mark(layer, "ffn_fwd")
    if mode == "local":
        out = ops.combine(Y, plan.dest_row, w, k)
        ret, row = Y, plan.dest_row
    elif scatter:
        yield (BARRIER, sym, torch.cuda.current_stream(dev))
        row = plan.slot                     # rows came back to their send slots
        out = ops.combine(Y, row, w, k)     # local reads only
        ret = Y
    elif mode == "p2p":
        yield (BARRIER, sym, torch.cuda.current_stream(dev))
        out = ops.combine_p2p(sym.peers(1), plan.dest_rank, plan.dest_row, w, k, d)
        ret, row = Y, plan.dest_row
    else:
        send_sizes, recv_counts, max_seg = sizes
        Yst = torch.empty((sum(recv_counts), d), dtype=torch.bfloat16, device=dev)
        ops.copy_segments(Y, Yst, plan.recv_src_off, plan.recv_stage_off, plan.recv_cnt,
                          max_seg)
        ret = torch.empty((P, d), dtype=torch.bfloat16, device=dev)
        yield (A2A, ret, Yst, send_sizes, recv_counts)
        out = ops.combine(ret, plan.slot, w, k)
        row = plan.slot
    _mark(layer, "combine")
    st.update(Tn=Tn, cap=cap, sizes=sizes, mode=mode, version=layer._fwd_version,
              self_rows=self_rows, plan=plan, idx=idx, w=w, probs=probs, off=off, X=X, H=H,
              A=A, ret=ret, row=row)
    return out


def _backward_steps(layer: MoELayer, st: dict, x, wg, w1, w2, dout):
    """One rank's backward; yields exchange requests and returns
    (dx, dwg, dbg, dW1, dW2) with the expert grads summed over their owner sets."""
    plan: DevicePlan = st["plan"]
    Tn, cap, sizes, mode = st["Tn"], st["cap"], st["sizes"], st["mode"]
    idx, w, probs, off, X, H, A, ret, row = (st[n] for n in
                                             ("idx", "w", "probs", "off", "X", "H", "A", "ret",
                                              "row"))
    k, N, rank = layer.k, layer.world, layer.rank
    d = layer.d
    G = len(layer.local_ids)
    dout = dout.contiguous().to(torch.bfloat16)
    _mark(layer, "bwd_start")
    dev = x.device
    scatter = mode == "p2p" and layer.scatter
    sym = None
    if mode == "local":
        dY = torch.empty((cap, d), dtype=torch.bfloat16, device=dev)
        dX = torch.empty((cap, d), dtype=torch.bfloat16, device=dev)
        dw = ops.combine_bwd(dout, ret, row, w, k, dY, plan.recv_m, plan.recv_off)
    elif mode == "p2p":
        if st["version"] != layer._fwd_version:
            raise RuntimeError("P2P exchange keeps one forward in flight per layer: "
                               "run backward before the next forward")
        sym = layer._symm
        dY, dX = sym.buf(2), sym.buf(3)
        if scatter:
            dw = ops.combine_bwd_p2p_ret(dout, ret, row, sym.peers(2), plan.dest_rank,
                                         plan.dest_row, w, k, dY, plan.recv_m, plan.recv_off)
            ops.signal_peers(sym.flag_peers[1], N, rank, sym.epoch)
            yield (SYNC,)
        else:
            dw = ops.combine_bwd_p2p(dout, sym.peers(1), sym.peers(2), plan.dest_rank,
                                     plan.dest_row, w, k, dY, plan.recv_m, plan.recv_off)
            yield (BARRIER, sym, torch.cuda.current_stream(dev))
    else:
        send_sizes, recv_counts, max_seg = sizes
        dret = torch.empty_like(ret)
        dw = ops.combine_bwd(dout, ret, row, w, k, dret)
        stage = torch.empty((sum(recv_counts), d), dtype=torch.bfloat16, device=dev)
        yield (A2A, stage, dret, recv_counts, send_sizes)
        dY = torch.empty((cap, d), dtype=torch.bfloat16, device=dev)
        dX = torch.empty((cap, d), dtype=torch.bfloat16, device=dev)
        ops.zero_pad_rows(dY, plan.recv_m, plan.recv_off)
        ops.copy_segments(stage, dY, plan.recv_stage_off, plan.recv_src_off, plan.recv_cnt,
                          max_seg)
        del dret, stage
    _mark(layer, "combine_bwd")
    main = torch.cuda.current_stream(dev)
    nx = layer.tail_overlap_nx if layer.tail_overlap_nx is not None else N >= 4
    tail = layer.tail_overlap and (mode == "local" or (scatter and nx))
    early = layer.early_router_wgrad and not tail
    side = None
    if early:
        if layer._tail_stream is None:
            layer._tail_stream = torch.cuda.Stream(dev)
        side = layer._tail_stream
        dlog_e = ops.gate_bwd(probs, idx, dw, layer.renorm)
        side.wait_stream(main)
        _mark(layer, "side_start", side)
        with torch.cuda.stream(side):
            dwg, dbg = ops.router_wgrad(dlog_e, x)
        _mark(layer, "router_wgrad", side)
    swi = layer.activation == "swiglu"
    dH = torch.empty_like(H)
    dW1 = torch.empty_like(w1)
    dW2 = torch.empty_like(w2)
    epi2 = _lib.LZ_EPI_DSWIGLU if swi else _lib.LZ_EPI_DGELU
    # while the replica-group all-reduces of the weight gradients run on NCCL's streams,
    # the GEMMs next to them leave `overlap_reserve` SMs free
    ov = max(2, (lzh_num_sms() - layer.overlap_reserve)) if N > 1 else 0
    # tail overlap (N = 1): dX GEMM right after the dgrad GEMM; the dispatch backward +
    # router weight gradient (they need only dX, dw and the gate state) then run on a side
    # stream under the two weight-gradient GEMMs.  N = 2, 3 keep the dX GEMM last, where it
    # hides the all-reduce of the last expert gradient, which the tail overlap would expose
    # instead; from N = 4 the exposed dispatch backward costs more (see tail_overlap_nx).
    if G > 0:
        # dA = dY . W2 (W2_e [d, d_ff] read MN-major), dH = dA * act'(H); on N > 1 the
        # tiles of our own rows start while the other ranks' dY rows arrive
        if scatter:
            ops.grouped_gemm_arrival(dY, w2, off, dH, st["self_rows"], sym.flags[1], sym.epoch,
                                     b_major=_lib.LZ_MN_MAJOR, aux=H, epilogue=epi2)
        else:
            ops.grouped_gemm_rows(dY, w2, off, dH, b_major=_lib.LZ_MN_MAJOR, aux=H,
                                  epilogue=epi2)
    works = []
    if tail:
        if G > 0:
            # dX = dH . W1 (W1_e [d_ff, d] read MN-major); scatter: rows go back to their
            # source ranks' return buffers (GEMM + dispatch-backward all-to-all fused)
            if scatter:
                ops.grouped_gemm_scatter(dH, w1, off, dX, sym.ret, sym.peers(3),
                                         sym.peers_host(3), sym.rows, b_major=_lib.LZ_MN_MAJOR)
            else:
                ops.grouped_gemm_rows(dH, w1, off, dX, b_major=_lib.LZ_MN_MAJOR)
        if layer._tail_stream is None:
            layer._tail_stream = torch.cuda.Stream(dev)
        side = layer._tail_stream
        side.wait_stream(main)
        _mark(layer, "side_start", side)
        if scatter:
            yield (BARRIER, sym, side)      # every owner's dX rows are back here
        with torch.cuda.stream(side):
            dx, dlog = ops.dispatch_bwd(dX, row, probs, idx, dw, wg, layer.renorm, Tn)
        _mark(layer, "dispatch_bwd", side)
        with torch.cuda.stream(side):
            dwg, dbg = ops.router_wgrad(dlog, x)
        _mark(layer, "router_wgrad", side)
    if G > 0:
        # variable-K weight gradients: dW1_e = dH_e^T X_e first -- the larger all-reduce
        # (2x for SwiGLU's W1|W3) then overlaps the next GEMM -- then dW2_e = dY_e^T A_e
        ops.grouped_gemm_wgrad(dH, X, off, dW1)
    if N > 1:
        works += (yield (EXPERT_AR, layer, [dW1])) or []
    if N > 1 and tail and layer.split_last_wgrad:
        # the last expert-gradient all-reduce is exposed with the tail overlap: the dW2 GEMM
        # runs as two launches split by expert id, so the first half's all-reduce overlaps
        # the second half's GEMM (same id split on every rank -> same request sequence)
        half = layer.E // 2
        ga = sum(1 for e in layer.local_ids if e < half)
        if ga > 0:
            ops.grouped_gemm_wgrad(dY, A, off[:ga + 1], dW2[:ga], num_sms=ov)
        works += (yield (EXPERT_AR, layer, [dW2], (0, half))) or []
        if G - ga > 0:
            ops.grouped_gemm_wgrad(dY, A, off[ga:], dW2[ga:], num_sms=ov)
        works += (yield (EXPERT_AR, layer, [dW2], (half, layer.E))) or []
    else:
        if G > 0:
            ops.grouped_gemm_wgrad(dY, A, off, dW2, num_sms=ov)
        if N > 1:
            works += (yield (EXPERT_AR, layer, [dW2])) or []
    if not tail:
        if G > 0:
            if scatter:
                ops.grouped_gemm_scatter(dH, w1, off, dX, sym.ret, sym.peers(3),
                                         sym.peers_host(3), sym.rows, b_major=_lib.LZ_MN_MAJOR,
                                         num_sms=ov)
            else:
                ops.grouped_gemm_rows(dH, w1, off, dX, b_major=_lib.LZ_MN_MAJOR, num_sms=ov)
    _mark(layer, "ffn_bwd")
    if tail:
        main.wait_stream(side)
        for t_ in (dx, dlog, dwg, dbg):
            if t_ is not None:
                t_.record_stream(main)
    else:
        if mode == "local" or scatter:
            if scatter:
                yield (BARRIER, sym, main)
            dx, dlog = ops.dispatch_bwd(dX, row, probs, idx, dw, wg, layer.renorm, Tn)
        elif mode == "p2p":
            yield (BARRIER, sym, main)
            dx, dlog = ops.dispatch_bwd_p2p(sym.peers(3), plan.dest_rank, plan.dest_row, probs,
                                            idx, dw, wg, layer.renorm, Tn, d)
        else:
            send_sizes, recv_counts, max_seg = sizes
            dXst = torch.empty((sum(recv_counts), d), dtype=torch.bfloat16, device=dev)
            ops.copy_segments(dX, dXst, plan.recv_src_off, plan.recv_stage_off, plan.recv_cnt,
                              max_seg)
            dxe = torch.empty((Tn * k, d), dtype=torch.bfloat16, device=dev)
            yield (A2A, dxe, dXst, send_sizes, recv_counts)
            dx, dlog = ops.dispatch_bwd(dxe, row, probs, idx, dw, wg, layer.renorm, Tn)
        _mark(layer, "dispatch_bwd")
        if early:
            main.wait_stream(side)
            for t_ in (dwg, dbg, dlog_e):
                if t_ is not None:
                    t_.record_stream(main)
        else:
            dwg, dbg = ops.router_wgrad(dlog, x)
            _mark(layer, "router_wgrad")
    if N > 1:
        yield (WAIT, works)
        flat = torch.cat([dwg.view(-1), dbg])
        yield (ALLREDUCE, flat)
        dwg = flat[:dwg.numel()].view_as(dwg)
        dbg = flat[dwg.numel():]
    _mark(layer, "grad_sync")
    return dx, dwg.to(wg.dtype), dbg, dW1, dW2


class _MoEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, wg, bg, w1, w2, layer: MoELayer):
        st: dict = {}
        if _NVTX:
            torch.cuda.nvtx.range_push("lz.moe_forward")
        out = layer.fabric.run(_forward_steps(layer, x, wg, bg, w1, w2, st))
        if _NVTX:
            torch.cuda.nvtx.range_pop()
        ctx.layer = layer
        ctx.st = st
        ctx.save_for_backward(x, wg, w1, w2)
        return out

    @staticmethod
    def backward(ctx, dout):
        x, wg, w1, w2 = ctx.saved_tensors
        layer: MoELayer = ctx.layer
        if _NVTX:
            torch.cuda.nvtx.range_push("lz.moe_backward")
        grads = layer.fabric.run(_backward_steps(layer, ctx.st, x.contiguous(), wg, w1, w2, dout))
        if _NVTX:
            torch.cuda.nvtx.range_pop()
        ctx.st = None
        return (*grads, None)


def run_step(layers, step_fn, max_reruns: int = 3):
    """Run one training step ``step_fn()`` (forward + backward through ``layers``), check
    every layer, and apply the exchange-capacity protocol: a plan that needs more exchange
    rows raises the same ExchangeCapacityError on every rank (nothing was exchanged), so
    every rank grows its buffers (``reserve``) and re-runs the step.  Returns step_fn's
    value of the successful run.  StepAbortedError (a lost peer) propagates."""
    from .dispatch import ExchangeCapacityError
    for attempt in range(max_reruns + 1):
        out = step_fn()
        torch.cuda.synchronize()
        try:
            for L in layers:
                L.check()
            return out
        except ExchangeCapacityError as exc:
            if attempt == max_reruns:
                raise
            for L in layers:
                L.reserve(exc.rows)
    raise AssertionError("unreachable")


def zipf_router_bias(n_experts: int, s: float, seed: int = 0) -> torch.Tensor:
    """log p_e with p_e ~ (1 + pi(e))^-s for a seeded permutation pi: makes the learned
    router's top-k a Zipf(s) sample (SURVEY.md 8d synthetic inputs)."""
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(n_experts, generator=g).float()
    p = (1.0 + perm) ** (-s)
    p = p / p.sum()
    return torch.log(p)


def default_slots(n_experts: int, n_ranks: int, factor: int = 3) -> int:
    """c = ceil(factor * E / N)."""
    return math.ceil(factor * n_experts / n_ranks)


__all__ = ["MoELayer", "StepAbortedError", "run_step", "zipf_router_bias", "default_slots"]
