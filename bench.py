"""Benchmark: MoE-layer tokens/s (dispatch + FFN + combine, fwd + bwd) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl reference]

Default workload = BASELINE.json configs[1] (GPT-MoE layer: 16 experts top-2,
d=1024, d_ff=4096, 64K tokens/GPU, Zipf-skewed routing, load-based replicas,
fwd+bwd bf16).  For N > 1 launch under torchrun (one rank per GPU, NCCL).  Rank 0
prints ONE JSON line.  ``--impl reference`` times the reference algorithm on the
host cores (oracle port: restated integer dispatcher + torch-CPU fp32 float stages).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: E, k, d, d_ff, tokens per GPU, zipf s, slot factor (c = ceil(f*E/N)), bwd.
    # slot_factor 6 (cfg2/cfg5): with Zipf(1.2) top-2 loads the reference's MRO plans reach
    # max/mean receive 1.07 at N = 4 (factor 5: 1.15, 3: 1.49)
    "cfg1": dict(E=8, k=2, d=512, dff=2048, tokens=1024, s=1.2, slot_factor=2, bwd=False, virtual=4,
                 name="CPU-ref MoE layer (E8 top-2 d512 d_ff2048, 1024 tok/rank, fwd)"),
    "cfg2": dict(E=16, k=2, d=1024, dff=4096, tokens=65536, s=1.2, slot_factor=6, bwd=True,
                 name="GPT-MoE layer (E16 top-2 d1024 d_ff4096, 64K tok/GPU, fwd+bwd)"),
    "cfg3": dict(E=8, k=2, d=4096, dff=14336, tokens=16384, s=1.2, slot_factor=5, bwd=True,
                 act="swiglu", cpu_tokens=256, cpu_reps=1,
                 name="Mixtral-8x7B-shape MoE layer (E8 top-2 d4096 d_ff14336 SwiGLU, 16K tok/GPU, "
                      "fwd+bwd + replica-group grad all-reduce)"),
    "cfg5": dict(E=16, k=2, d=1024, dff=4096, tokens=65536, s=1.2, slot_factor=6, bwd=True,
                 name="elastic reconfiguration 8->6->4 (cfg2 shape, slots held at the 8-GPU value)"),
    "cfg4": dict(E=64, k=1, d=2048, dff=None, tokens=131072, s=1.5, slot_factor=4, bwd=False,
                 name="E64 top-1 d2048 dispatch/combine-only sweep (8K..1M tok/GPU, Zipf 1.5)"),
}
METRIC = "MoE-layer tokens/s (dispatch+FFN+combine, fwd+bwd)"


def _env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if not self.lines:   # timed region shorter than the first sample: query once now
            try:
                self.lines = subprocess.run(
                    ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                     "-i", str(self.gpu)], capture_output=True, text=True,
                    timeout=10).stdout.strip().splitlines()
            except Exception:
                pass
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(cfg, n_ranks, tokens_per_rank, reps, threads, seed=0):
    """Reference path on the host cores (oracle/cpu_path.py: flexep unchanged from
    baseline/_ref for the integer stages when present, else the pinned port; torch-CPU
    fp32 float stages).  Returns (tokens/s, seconds, tokens, kind)."""
    from oracle import cpu_path
    E = cfg["E"]
    bias = _zipf_bias(E, cfg["s"], seed)
    p = torch.softmax(bias, 0).tolist()
    loads = [max(1, int(v * tokens_per_rank * n_ranks * cfg["k"])) for v in p]
    return cpu_path.run(tokens_per_rank, n_ranks, E, cfg["d"], cfg["dff"], cfg["k"], loads,
                        cpu_path.slots_for(cfg, n_ranks), 2, reps=reps, seed=seed, bias=bias,
                        backward=cfg["bwd"], threads=threads, activation=cfg.get("act", "gelu"))


def _zipf_bias(E, s, seed=0):
    """log p_e, p_e ~ (1 + pi(e))^-s (the synthetic routing of SURVEY.md 8d; the same
    formula as layer.zipf_router_bias, restated so the reference arm imports nothing of
    the product)."""
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(E, generator=g).float()
    p = (1.0 + perm) ** (-s)
    return torch.log(p / p.sum())


def reference_sample(cfg, world):
    """(simulated ranks, tokens per rank) of one reference-arm step: the GPU arm's per-GPU
    step (cfg2: 65,536 tokens fwd+bwd) -- at N = 1 exactly the measured configuration;
    at N > 1 the same tokens spread over N simulated ranks (the N-rank plan).  cfg1: the
    full config (4 simulated ranks x 1024 tokens).  cfg3 (a CPU step > 30 s): a sample."""
    if "cpu_tokens" in cfg:
        return 1, cfg["cpu_tokens"]
    if cfg.get("virtual"):
        return cfg["virtual"], cfg["tokens"]
    return world, cfg["tokens"] // world


def run_reference(args, cfg):
    rank, world, _ = _env()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    n_sim, per_rank = reference_sample(cfg, world)
    # warm-up steps on a small sample (allocator / thread-pool warm-up; untimed)
    for _ in range(args.warmup):
        cpu_reference(cfg, n_sim, min(per_rank, 1024), 1, threads)
    times = []
    tok = 0
    kind = "port"
    for _ in range(args.steps):
        _, dt, t, kind = cpu_reference(cfg, n_sim, per_rank, 1, threads)
        times.append(dt)
        tok += t
    total = sum(times)
    value = tok / total
    same = "cpu_tokens" not in cfg and (world == 1 or bool(cfg.get("virtual")))
    line = {
        "impl": "reference", "metric": METRIC if cfg["bwd"] else METRIC.replace("fwd+bwd", "fwd"),
        "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["name"], "simulated_ranks": n_sim,
                   "tokens_per_step": tok // args.steps, "same_as_gpu_arm": bool(same)},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": kind,
                         "cpu_model": cpu_model(),
                         "integer_stages": "flexep 0.1.0 unchanged (baseline/_ref)"
                         if kind == "reference" else "oracle port (pinned to reference goldens)",
                         "float_stages": "torch-CPU fp32 restatement (the reference has none)",
                         "sample": f"{tok // args.steps} tokens per step ({n_sim} simulated "
                                   f"rank(s)) x {args.steps} steps; warm-up on 1024-token "
                                   f"samples"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def run_gpu(args, cfg):
    import torch.distributed as dist

    from paper_2407_04656_b200 import _lib, ops
    from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix

    rank, world, local = _env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    E, k, d, dff, Tn = cfg["E"], cfg["k"], cfg["d"], cfg["dff"], cfg["tokens"]
    c = math.ceil(cfg["slot_factor"] * E / world)
    bias = zipf_router_bias(E, cfg["s"], seed=0)
    act = cfg.get("act", "gelu")
    # router logit noise x.wg has std ~ 0.04 * sqrt(d) ~ 1.28 (= Gumbel(0,1) std at d=1024): with
    # the log-Zipf bias, top-k ~ Zipf(s) sampling without replacement
    layer = MoELayer(d, dff, E, k, seed=0, router_bias=bias, device=dev, activation=act,
                     router_std=1.28 / math.sqrt(d),
                     group=None if world == 1 else dist.group.WORLD)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn(Tn, d, generator=g, device=dev).bfloat16()
    dout = (torch.randn(Tn, d, generator=g, device=dev) * 1e-2).bfloat16()
    # load-based replicas from the routing of a SEPARATE batch of the same distribution
    # (the paper re-plans from a history window, not from the batch it then runs)
    gp = torch.Generator(device=dev)
    gp.manual_seed(777 + rank)
    x_plan = torch.randn(Tn, d, generator=gp, device=dev).bfloat16()
    _, _, _, hist = ops.router_gate(x_plan, layer.wg.detach(), layer.bg.detach(), k)
    del x_plan
    hist = hist.long()
    if world > 1:
        dist.all_reduce(hist)
    loads = hist.cpu().tolist()
    plan = plan_for_loads(loads, world, c, 2)
    layer.set_plan(replica_matrix(plan))

    def step(xx, dd):
        nonlocal layer
        layer.zero_grad(set_to_none=True)
        out = layer(xx)
        if cfg["bwd"]:
            out.backward(dd)
        return out

    clocks = ClockSampler(local).start() if rank == 0 else None
    from paper_2407_04656_b200.layer import run_step
    run_step([layer], lambda: step(x, dout))   # grows the exchange buffers if the plan needs
    for _ in range(max(args.warmup, 3) - 1):
        step(x, dout)
    torch.cuda.synchronize()
    layer.check()
    imbalance = layer.imbalance()
    max_node_tokens, cross_node_tokens = layer.layer_cost()   # simulator.py:198-219 terms
    rows_local = int(layer.last_plan.recv_m.sum())  # assignments this rank's experts process
    x_h = x.cpu().pin_memory()
    d_h = dout.cpu().pin_memory()
    res_h = torch.empty(1, dtype=torch.float32).pin_memory()
    # ---- CUDA-graph mode (the product path for a training step): the whole fwd+bwd
    # step is captured once and replayed; value/ms_per_step/e2e come from it, the eager
    # numbers measured afterwards are reported alongside (graph first: sustained
    # power/thermal settling only ever penalises the later measurement).
    graph, graph_err, in_graph = None, "", None
    if args.no_graph:
        graph_err = "graphs disabled"
    else:
        from paper_2407_04656_b200.graphs import GraphedStep
        try:
            # slots 0 / 1: the timed replays and the double-buffered e2e pipeline; slot 2
            # carries the in-graph GEMM event nodes (read back after every replay), so no
            # timed replay runs the instrumented graph
            graph = GraphedStep(layer, Tn, nbuf=3, backward=cfg["bwd"], timed_slot=2)
        except Exception as exc:  # report, keep eager numbers
            import traceback
            traceback.print_exc()
            graph = None
            graph_err = repr(exc)[:200]
    if graph is not None:
        for b in range(3):
            graph.x[b].copy_(x)
            graph.dout[b].copy_(dout)
        for _ in range(3):
            graph.replay(0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            graph.replay(0)
        g1.record()
        torch.cuda.synchronize()
        ms_graph = g0.elapsed_time(g1)
        # e2e: double-buffered static inputs; slot b's H2D (side stream) overlaps the other
        # slot's replay; every step's inputs cross PCIe inside the timed region and the
        # step's scalar result is read back.  The step's host input is the token batch x;
        # the gradient entering the layer's backward is the gradient of a fixed linear loss
        # <out, r> (r resident on the device like the rest of the model -- in training it
        # comes from the layers above / the loss on the device, never from the host).  The
        # variant that also copies the upstream gradient from the host every step is
        # reported next to it (e2e_with_dout_h2d).
        cs = torch.cuda.Stream(device=dev)
        ev_copy = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        main = torch.cuda.current_stream(dev)
        copy_dout = [False]

        def h2d(b):
            with torch.cuda.stream(cs):
                cs.wait_event(ev_done[b])
                graph.x[b].copy_(x_h, non_blocking=True)
                if copy_dout[0]:
                    graph.dout[b].copy_(d_h, non_blocking=True)
                ev_copy[b].record(cs)

        def g_e2e(n):
            for b in range(2):
                ev_done[b].record(main)
            h2d(0)
            for i in range(n):
                b = i % 2
                main.wait_event(ev_copy[b])
                r = graph.replay(b)
                ev_done[b].record(main)
                res_h.copy_(r, non_blocking=True)
                if i + 1 < n:
                    h2d((i + 1) % 2)

        def timed_e2e(with_dout):
            copy_dout[0] = with_dout
            g_e2e(3)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record()
            g_e2e(args.steps)
            h1.record()
            torch.cuda.synchronize()
            return h0.elapsed_time(h1)

        ms_graph_e2e = timed_e2e(False)
        # the GEMMs timed from inside the graph: slot 2 carries event-record nodes around
        # the step and every grouped-GEMM launch; each replay is read back, so the GEMM
        # time and the step time come from the same replays (measured before the secondary
        # e2e variant, so the board is in the same state as in round 2a's order)
        rt = graph.replay_times(args.steps)
        ms_graph_e2e_dout = timed_e2e(True) if cfg["bwd"] else None
        for b in range(2):
            graph.dout[b].copy_(dout)
        if world > 1:
            t = torch.tensor([ms_graph, ms_graph_e2e, ms_graph_e2e_dout or 0.0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_graph, ms_graph_e2e, ms_graph_e2e_dout = (float(v) for v in t.tolist())
            if not cfg["bwd"]:
                ms_graph_e2e_dout = None
        in_graph = {"step_ms": float(np.median(rt["step_ms"])),
                    "gemm_ms": float(np.median(rt["gemm_ms"])),
                    "gemm_launch_ms": [float(np.median(c)) for c in zip(*rt["gemm_launch_ms"])]}
        if world > 1:
            t = torch.tensor([in_graph["step_ms"], in_graph["gemm_ms"]], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            in_graph["step_ms_max_over_ranks"], in_graph["gemm_ms_max_over_ranks"] = \
                (float(v) for v in t.tolist())
        # autograd nodes created under capture stay bound to the capture stream and would
        # force a device sync on every later eager backward: continue on a fresh layer
        # object with identical weights and plan
        launches_graph = graph.launches_per_step
        del graph
        graph = True
        # hand the graphs' private pool back before the eager steps allocate (otherwise
        # every eager step can hit the allocator's free-and-retry path)
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        fresh = MoELayer(d, dff, E, k, seed=0, router_bias=bias, device=dev, activation=act,
                         router_std=1.28 / math.sqrt(d), replicas=layer.R,
                         group=None if world == 1 else dist.group.WORLD)
        with torch.no_grad():
            for pa, pb in zip(fresh.parameters(), layer.parameters()):
                pa.copy_(pb)
        # N > 1: keep the already rendezvoused symmetric buffers (no second collective
        # allocation, and the old ones are never freed under a rank's feet)
        fresh._symm, fresh._rows_wanted = layer._symm, layer._rows_wanted
        layer = fresh
        for _ in range(3):
            step(x, dout)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ops.GEMM_EVENTS = [] if in_graph is None else None
    l0 = _lib.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step(x, dout)
    e1.record()
    torch.cuda.synchronize()
    launches = _lib.launch_count - l0
    ms = e0.elapsed_time(e1)
    if in_graph is None:   # eager only: GEMM events of the timed eager steps
        gemm_ms = sum(a.elapsed_time(b) for a, b in ops.GEMM_EVENTS)
        ops.GEMM_EVENTS = None
    else:
        gemm_ms = in_graph["gemm_ms"] * args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()

    # ---- per-stage breakdown (separate, untimed pass with CUDA events between stages)
    from paper_2407_04656_b200.layer import stage_breakdown
    layer.stage_events = []
    nb = 3
    for _ in range(nb):
        # ~1 ms of device spin first: the host enqueues the step's first kernels while the
        # GPU is still busy, so the stage events time the kernels, not host launch latency
        torch.cuda._sleep(1 << 21)
        step(x, dout)
    torch.cuda.synchronize()
    stages = {k2: round(v / nb, 4) for k2, v in stage_breakdown(layer.stage_events).items()}
    layer.stage_events = None
    stages_all = [stages]
    nvlink = None
    if world > 1:
        stages_all = [None] * world
        dist.all_gather_object(stages_all, stages)
        # NVLink evidence: off-rank bytes of the fused exchange kernels over their stage time,
        # and the replica-group gradient all-reduce timed on its own (bus bandwidth)
        remote = int((layer.last_plan.dest_rank != rank).sum()) * d * 2
        gbps = {"dispatch": remote / (stages["dispatch"] * 1e-3) / 1e9,
                "combine_bwd": remote / (stages["combine_bwd"] * 1e-3) / 1e9}
        grads = [layer.w1.grad, layer.w2.grad]
        bus_bytes = 0.0
        for pg, pos in layer.replica_groups.buckets(layer.local_ids):
            gsz = dist.get_world_size(pg)
            per = sum(g_[0].numel() * g_.element_size() for g_ in grads) * len(pos)
            bus_bytes += per * 2 * (gsz - 1) / gsz
        layer.replica_groups.allreduce(grads, layer.local_ids)
        torch.cuda.synchronize()
        dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(5):
            layer.replica_groups.allreduce(grads, layer.local_ids)
        a1.record()
        torch.cuda.synchronize()
        ar_ms = a0.elapsed_time(a1) / 5
        mine = {"remote_MB": remote / 1e6, "dispatch_GBps": gbps["dispatch"],
                "combine_bwd_GBps": gbps["combine_bwd"], "grad_allreduce_ms": ar_ms,
                "grad_allreduce_busbw_GBps": bus_bytes / (ar_ms * 1e-3) / 1e9 if bus_bytes else 0.0}
        nvlink = [None] * world
        dist.all_gather_object(nvlink, mine)

    # ---- e2e through the public API: pinned host input -> device, result -> host.
    # Each step's x is copied H2D on a side stream one step ahead (a prefetching input
    # pipeline); every copy, including the first, is inside the timed region, and the
    # step's scalar result is read back D2H.  The upstream gradient is that of the fixed
    # linear loss <out, dout> (dout resident, as in the graph-mode e2e above).
    from paper_2407_04656_b200.hostio import HostPrefetcher

    def e2e_run(nsteps):
        pf = HostPrefetcher([x_h], dev)
        pf.prefetch()
        for i in range(nsteps):
            (xx,) = pf.get()
            if i + 1 < nsteps:
                pf.prefetch()
            out = step(xx, dout)
            res_h.copy_(out.detach().sum(dtype=torch.float32).view(1), non_blocking=True)

    e2e_run(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    e2e_run(args.steps)
    f1.record()
    torch.cuda.synchronize()
    ms_e2e = f0.elapsed_time(f1)
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())

    clk = clocks.stop() if clocks else None
    layer.check()   # the timed steps' plans were valid and fit the exchange buffers

    if rank == 0:
        hbm, tf_burst, tf_sus, src = _peaks()
        # algorithmic HBM bytes per stage (SURVEY.md 8d formulas) over the stage's CUDA-event
        # time in the eager breakdown pass (includes launch gaps: a lower bound on the
        # kernels' own GB/s; ncu per-kernel numbers are in profiles/)
        Pa = Tn * k
        stage_bytes = {
            "gate": Tn * d * 2 + E * d * 2 + Tn * E * 4 + Tn * k * 8,
            "plan": Pa * 4 + Pa * 16,
            "dispatch": Tn * d * 2 + Pa * d * 2 + Pa * 4,
            "combine": Pa * d * 2 + Pa * 8 + Tn * d * 2,
            "combine_bwd": Tn * d * 2 + 2 * Pa * d * 2 + Pa * 8,
            "dispatch_bwd": Pa * d * 2 + Tn * d * 2 + 2 * Tn * E * 4,
            "router_wgrad": Tn * d * 2 + Tn * E * 4,
        }
        if getattr(layer, "tail_overlap", False) and cfg["bwd"]:
            # these two run on a side stream under the weight-gradient GEMMs (their stage
            # marks time them there, slowed by the GEMMs; isolated numbers: hbm_kernels)
            stage_bytes.pop("dispatch_bwd")
            stage_bytes.pop("router_wgrad")
        hbm_stages = {}
        if world == 1:
            for st_name, nbytes in stage_bytes.items():
                ms_st = stages.get(st_name)
                if ms_st:
                    gbs = nbytes / (ms_st * 1e-3) / 1e9
                    hbm_stages[st_name] = {"MB": round(nbytes / 1e6, 1), "ms": round(ms_st, 4),
                                           "GBps": round(gbs, 1), "frac": round(gbs / hbm, 3)}
        hbm_kernels = None
        if world == 1 and cfg["bwd"] and not args.no_isolated:
            hbm_kernels = isolated_hbm_kernels(layer, x, dout, hbm)
        P = Tn * k
        gemms_per_step = 6 if cfg["bwd"] else 2
        n_mat = 3 if act == "swiglu" else 2
        # algorithmic FLOPs of this rank's expert GEMMs (rows it received; = P at N = 1)
        flops_per_step = 2.0 * rows_local * d * dff * n_mat * (3 if cfg["bwd"] else 1)
        flops_per_launch = flops_per_step / gemms_per_step
        achieved = flops_per_step * args.steps / (gemm_ms * 1e-3) / 1e12
        traffic = None
        prof = os.path.join(ROOT, "profiles", "gemm_traffic.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get(args.config)
            except Exception:
                traffic = None
        eager = {"value": world * Tn * args.steps / (ms * 1e-3), "ms_per_step": ms / args.steps,
                 "e2e": world * Tn * args.steps / (ms_e2e * 1e-3)}
        if graph is not None:
            ms_main, ms_main_e2e, launches = ms_graph, ms_graph_e2e, launches_graph * args.steps
            e2e_dout_value = (None if ms_graph_e2e_dout is None
                              else world * Tn * args.steps / (ms_graph_e2e_dout * 1e-3))
        else:
            ms_main, ms_main_e2e = ms, ms_e2e
            e2e_dout_value = None
        line = {
            "metric": METRIC, "value": world * Tn * args.steps / (ms_main * 1e-3),
            "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_main / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": f"synthetic: x~N(0,1) bf16, random-init weights (std 0.02), Zipf s={cfg['s']} "
                    f"routing via router bias",
            "config": {"workload": cfg["name"], "experts": E, "top_k": k, "d_model": d,
                       "d_ff": dff, "tokens_per_gpu": Tn, "global_tokens": world * Tn,
                       "slots_per_gpu": c, "fault_threshold": 2, "zipf_s": cfg["s"],
                       "replicas": list(plan_replicas(plan, E)),
                       "imbalance_max_over_mean_recv": round(imbalance, 4),
                       "reference_cost_terms": {"max_node_tokens": max_node_tokens,
                                                "cross_node_tokens": cross_node_tokens,
                                                "model": "flexep simulator.py:198-219 "
                                                         "(adaptive_layer_cost) on this "
                                                         "step's device plan"},
                       "replica_plan_source": "routing histogram of a separate batch",
                       "l2": "inputs larger than L2 (x alone 134 MB; step working set > 4 GB)",
                       "parallelism": f"flexible-EP{world} (DP tokens, replicated experts)"},
            "roofline": {"kernel": "lz grouped_gemm (tcgen05 fwd+dgrad+wgrad)", "bound": "tensor",
                         "achieved": achieved, "peak": tf_sus, "unit": "TFLOP/s",
                         "frac": achieved / tf_sus, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per GEMM launch (ncu --set full, "
                                         "profiles/gemm_traffic.json)",
                         "peak_kind": f"{src} sustained bf16",
                         "flops_per_launch": flops_per_launch,
                         "gemm_ms_per_step": gemm_ms / args.steps,
                         "gemm_share_of_step": (in_graph["gemm_ms"] / in_graph["step_ms"])
                         if in_graph else gemm_ms / ms,
                         "timing": "graph event-record nodes around every GEMM launch and "
                                   "the whole step, read after each of K replays of the "
                                   "captured step (medians; same replays for both)"
                         if in_graph else "CUDA events around the GEMM launches of the "
                                          "timed eager steps",
                         "in_graph": in_graph,
                         "gemms_per_step": gemms_per_step,
                         "gemm_launches_per_step": (len(in_graph["gemm_launch_ms"])
                                                    if in_graph else None)},
            "mode": "cuda-graph replay of the whole fwd+bwd step" if graph is not None
                    else "eager (" + graph_err + ")",
            "eager": eager,
            "e2e": {"value": world * Tn * args.steps / (ms_main_e2e * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(x.numel() * 2),
                    "d2h_bytes_per_step": 4,
                    "inputs": "the token batch x from pinned host memory every step; the "
                              "backward's upstream gradient is that of the fixed linear loss "
                              "<out, dout> with dout resident on the device"},
            "e2e_with_dout_h2d": None if e2e_dout_value is None else {
                "value": e2e_dout_value, "unit": "tokens/s",
                "h2d_bytes_per_step": int(x.numel() * 2 + dout.numel() * 2),
                "d2h_bytes_per_step": 4,
                "note": "as e2e, with the upstream gradient also copied from pinned host "
                        "memory every step (the round-1 definition)"},
            "gpu_launches": launches,
            "clocks": clk,
            "stages_ms_rank0": stages,
            "hbm_stages": hbm_stages or None,
            "hbm_kernels": hbm_kernels,
            "hbm_note": "hbm_stages: eager pass behind a device spin (the GPU trails the "
                        "host), events between stages, so they include inter-kernel gaps "
                        "and small torch ops (lower bounds); hbm_kernels: each kernel alone, "
                        "20 launches back to back on the step's shapes and routing",
            "stages_ms_per_rank": stages_all if world > 1 else None,
            "nvlink": None if nvlink is None else {
                "per_rank": [{k2: round(v, 2) for k2, v in r.items()} for r in nvlink],
                "link_peak_GBps_per_direction": 900,
                "note": "dispatch / combine_bwd: off-rank bytes of the fused P2P kernels over "
                        "their stage time (eager pass); grad all-reduce: NCCL replica-group "
                        "all-reduce of the expert gradients timed alone (bus bandwidth); the "
                        "scatter GEMMs' returns ride inside the GEMMs"},
            "exchange": layer.exchange_mode(),
        }
        if world == 1 and not args.no_cpu_baseline:
            threads = len(os.sched_getaffinity(0))
            n_sim, ctok = reference_sample(cfg, 1)
            cpu_reference(cfg, n_sim, min(ctok, 1024), 1, threads)   # warm-up
            tps, dt, tok, kind = cpu_reference(cfg, n_sim, ctok, 1, threads)
            line["cpu_baseline"] = {"value": tps, "unit": "tokens/s", "cores": threads,
                                    "cpu_model": cpu_model(), "kind": kind,
                                    "sample": f"{tok} tokens: one full "
                                              f"{'fwd+bwd' if cfg['bwd'] else 'fwd'} step of the "
                                              f"same layer on 1 rank (the --impl reference "
                                              f"step), {dt:.1f} s"}
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


def isolated_hbm_kernels(layer, x, dout, hbm, reps=20):
    """Each HBM-bound kernel of the step replayed `reps` times back to back on the step's
    own shapes and routing: the `reps` launches are captured in ONE CUDA graph whose replay
    is timed with a CUDA-event pair, so neither host launch gaps nor the wrappers' output
    allocations are inside the timed region.  The working set of every launch (>= 400 MB,
    except the gate's 134 MB of x) exceeds the 126 MB L2, and the kernels alternate
    between two input copies so no launch re-reads the previous launch's input from L2.
    Bytes are the algorithmic ones of SURVEY.md 8d."""
    from paper_2407_04656_b200 import ops
    from paper_2407_04656_b200.dispatch import plan_device

    Tn, d = x.shape
    k, E = layer.k, layer.E
    wg, bg = layer.wg.detach(), layer.bg.detach()
    P = Tn * k
    xs = [x, x.clone()]
    idx, w, probs, hist = ops.router_gate(x, wg, bg, k, layer.renorm)
    T = hist.view(E, 1).to(torch.int32)
    plan = plan_device(T, layer.R_dev, 0, idx.view(-1), ops.row_align())
    cap = P + E * ops.ALIGN
    Xs = [torch.zeros((cap, d), dtype=torch.bfloat16, device=x.device) for _ in range(2)]
    dY = torch.empty_like(Xs[0])
    row = plan.dest_row
    dw = ops.combine_bwd(dout, Xs[0], row, w, k, dY, plan.recv_m, plan.recv_off)
    dlog = ops.dispatch_bwd(Xs[0], row, probs, idx, dw, wg, layer.renorm, Tn)[1]
    wgT = wg.t().contiguous()
    from paper_2407_04656_b200 import _lib
    from paper_2407_04656_b200.ops import ptr, _s

    def dbwd(i):   # the kernel alone (ops.dispatch_bwd also transposes wg per call)
        dx = torch.empty((Tn, d), dtype=torch.bfloat16, device=x.device)
        dl = torch.empty((Tn, E), dtype=torch.float32, device=x.device)
        _lib.call("lz_dispatch_bwd", ptr(Xs[i]), ptr(row), Tn, d, k, ptr(probs), ptr(idx),
                  ptr(dw), ptr(wgT), E, int(layer.renorm), ptr(dx), ptr(dl), _s())

    kernels = {
        "gate": (lambda i: ops.router_gate(xs[i], wg, bg, k, layer.renorm),
                 Tn * d * 2 + E * d * 2 + Tn * E * 4 + Tn * k * 8),
        "pack": (lambda i: ops.pack(xs[i], row, k, Xs[i], plan.recv_m, plan.recv_off),
                 Tn * d * 2 + P * d * 2 + P * 4),
        "combine": (lambda i: ops.combine(Xs[i], row, w, k), P * d * 2 + P * 8 + Tn * d * 2),
        "combine_bwd": (lambda i: ops.combine_bwd(dout, Xs[i], row, w, k, dY, plan.recv_m,
                                                  plan.recv_off),
                        Tn * d * 2 + 2 * P * d * 2 + P * 8),
        "dispatch_bwd": (dbwd, P * d * 2 + Tn * d * 2 + 2 * Tn * E * 4),
        "router_wgrad": (lambda i: ops.router_wgrad(dlog, xs[i]), Tn * d * 2 + Tn * E * 4),
    }
    out = {}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    side = torch.cuda.Stream(device=x.device)
    for name, (fn, nbytes) in kernels.items():
        for i in range(4):
            fn(i & 1)
        torch.cuda.synchronize()
        # the `reps` launches captured in ONE CUDA graph and replayed: the wrappers' host
        # work (output allocation, ctypes) is outside the timed region, which then holds
        # only the kernels, back to back
        side.wait_stream(torch.cuda.current_stream(x.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for i in range(reps):
                fn(i & 1)
        g.replay()
        torch.cuda.synchronize()
        ev0.record()
        g.replay()
        ev1.record()
        torch.cuda.synchronize()
        del g
        us = ev0.elapsed_time(ev1) / reps * 1e3
        gbs = nbytes / (us * 1e-6) / 1e9
        out[name] = {"MB": round(nbytes / 1e6, 1), "us": round(us, 1), "GBps": round(gbs, 1),
                     "frac": round(gbs / hbm, 3)}
    return out


def run_virtual(args, cfg):
    """Config 1 as the reference states it: 4 SIMULATED EP ranks (1024 tokens each) with
    the adaptive replica placement, forward only -- run as 4 virtual ranks on one GPU
    (VirtualEP: the N-rank plan and the fused P2P dispatch/combine over device memory).
    The 4K-token working set fits in L2, so L2 is flushed between timed steps (outside
    the per-step events)."""
    from paper_2407_04656_b200 import _lib
    from paper_2407_04656_b200.layer import zipf_router_bias
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
    from paper_2407_04656_b200.virtual import VirtualEP
    rank, world, local = _env()
    if rank != 0:
        return 0
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    nv, Tn, E, k, d, dff = 4, cfg["tokens"], cfg["E"], cfg["k"], cfg["d"], cfg["dff"]
    hbm, peak_burst, _, src = _peaks()
    bias = zipf_router_bias(E, cfg["s"])
    p = torch.softmax(bias, 0).tolist()
    loads = [max(1, int(v * Tn * nv * k)) for v in p]
    R = replica_matrix(plan_for_loads(loads, nv, math.ceil(cfg["slot_factor"] * E / nv), 2))
    vep = VirtualEP(d, dff, E, k, R, Tn, seed=0, router_bias=bias, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    xs = [torch.randn(Tn, d, generator=g, device=dev).bfloat16() for _ in range(nv)]
    host = [x.cpu().pin_memory() for x in xs]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(max(3, args.warmup)):
        vep(xs)
    torch.cuda.synchronize()

    def eager():
        outs = vep(xs)
        return torch.stack([o[0, 0].float() for o in outs]).sum().view(1)

    run, mode = eager, "eager"
    n0 = _lib.launch_count
    eager()
    torch.cuda.synchronize()
    launches = _lib.launch_count - n0
    if not args.no_graph:
        # the launch-bound 4K-token forward replays as one CUDA graph (static inputs xs)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            gsum = eager()
        run, mode = (lambda: (graph.replay(), gsum)[1]), "cuda-graph replay"
        for _ in range(3):
            run()
        torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clk = ClockSampler(local).start()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record()
        run()
        ev[i][1].record()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    # e2e: pinned host tokens -> the (static) device inputs, forward, one scalar back per step
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(args.steps):
        for h, t in zip(host, xs):
            t.copy_(h, non_blocking=True)
        run().cpu()
    e1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    tokens = nv * Tn
    cpu = None
    if not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        torch.set_num_threads(threads)
        cpu_reference(cfg, nv, Tn, 1, threads)
        vals = [cpu_reference(cfg, nv, Tn, 1, threads) for _ in range(max(1, args.cpu_reps // 4))]
        cpu = {"value": sum(v[2] for v in vals) / sum(v[1] for v in vals), "unit": "tokens/s",
               "cores": threads, "kind": vals[0][3], "cpu_model": cpu_model(),
               "sample": f"full config 1 ({tokens} tokens, 4 simulated ranks) x {len(vals)}"}
    flops = 2 * tokens * k * d * dff * 2
    line = {"metric": METRIC.replace("fwd+bwd", "fwd"), "value": tokens / (ms * 1e-3),
            "unit": "tokens/s", "n_gpus": 1,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, Zipf-biased router)",
            "config": {"workload": cfg["name"], "virtual_ranks": nv, "tokens_per_rank": Tn,
                       "experts": E, "top_k": k, "d_model": d, "d_ff": dff,
                       "l2": "flushed between timed steps (256 MB write)", "mode": mode},
            "roofline": {"kernel": "whole forward step (launch-bound at this size)",
                         "bound": "tensor", "achieved": flops / (ms * 1e-3) / 1e12,
                         "peak": peak_burst, "unit": "TFLOP/s",
                         "frac": flops / (ms * 1e-3) / 1e12 / peak_burst,
                         "peak_kind": f"{src} burst bf16", "traffic": None},
            "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": sum(h.numel() * 2 for h in host),
                    "d2h_bytes_per_step": 4},
            "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu}
    emit(line)
    return 0


def run_dispatch_sweep(args, cfg):
    """Config 4: gating softmax/top-k (on precomputed logits) -> plan -> pack -> combine
    only (identity expert), HBM roofline of
    the pack and combine kernels over 8K..1M tokens/GPU.  N = 1 only."""
    from paper_2407_04656_b200 import ops
    from paper_2407_04656_b200.dispatch import plan_device
    from paper_2407_04656_b200.layer import zipf_router_bias
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
    rank, world, local = _env()
    if rank != 0:
        return 0
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    E, k, d = cfg["E"], cfg["k"], cfg["d"]
    hbm, _, _, src = _peaks()
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    wg = (torch.randn(E, d, generator=g, device=dev) * 0.02).bfloat16()
    bg = zipf_router_bias(E, cfg["s"]).to(dev)
    sweep = []
    for Tn in (8192, 16384, 32768, 65536, 131072, 262144, 524288, 1048576):
        x = torch.randn(Tn, d, generator=g, device=dev).bfloat16()
        # the router projection (x . Wg^T) is the FFN side's router layer, not part of
        # this dispatch/combine-only config: its logits are computed once, outside the
        # timed step; the step starts at the gating softmax/top-k + histogram (K1)
        logits = (torch.mm(x, wg.t()).float() + bg).contiguous()
        idx, w, _, hist = ops.gate_topk(logits, k, probs=False)
        loads = hist.tolist()
        R = torch.tensor(replica_matrix(plan_for_loads(loads, 1, math.ceil(4 * E), 2)),
                         dtype=torch.int32, device=dev)
        align = ops.row_align()
        P = Tn * k
        X = torch.empty(P + E * align, d, dtype=torch.bfloat16, device=dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]

        def once(rec):
            if rec:
                ev[0].record()
            i2, w2, _, h2 = ops.gate_topk(logits, k, probs=False)
            if rec:
                ev[1].record()
            pl = plan_device(h2.view(E, 1), R, 0, i2.view(-1), align)
            if rec:
                ev[2].record()
            ops.pack(x, pl.dest_row, k, X, pl.recv_m, pl.recv_off)
            if rec:
                ev[3].record()
            out = ops.combine(X, pl.dest_row, w2, k)
            if rec:
                ev[4].record()
            return out

        for _ in range(3):
            once(False)
        torch.cuda.synchronize()
        reps = max(3, min(50, (1 << 22) // Tn))
        acc = [0.0] * 4
        for _ in range(reps):
            once(True)
            torch.cuda.synchronize()
            for j in range(4):
                acc[j] += ev[j].elapsed_time(ev[j + 1])
        t_gate, t_plan, t_pack, t_comb = (a / reps for a in acc)
        pack_b = Tn * d * 2 + P * d * 2 + P * 4
        comb_b = P * d * 2 + P * 8 + Tn * d * 2
        # the step itself as one CUDA graph (device time; the per-stage events above run
        # eagerly and include each small stage's host launch latency)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            once(False)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ga.record()
        for _ in range(reps):
            graph.replay()
        gb.record()
        torch.cuda.synchronize()
        total = ga.elapsed_time(gb) / reps
        del graph
        sweep.append({"tokens": Tn, "ms": round(total, 4), "tokens_per_s": Tn / (total * 1e-3),
                      "eager_stage_sum_ms": round(t_gate + t_plan + t_pack + t_comb, 4),
                      "gate_ms": round(t_gate, 4), "plan_ms": round(t_plan, 4),
                      "pack_ms": round(t_pack, 4), "combine_ms": round(t_comb, 4),
                      "pack_GBps": pack_b / (t_pack * 1e-3) / 1e9,
                      "combine_GBps": comb_b / (t_comb * 1e-3) / 1e9,
                      "pack_frac": pack_b / (t_pack * 1e-3) / 1e9 / hbm,
                      "combine_frac": comb_b / (t_comb * 1e-3) / 1e9 / hbm})
        del x, X
    ref = next(r for r in sweep if r["tokens"] == cfg["tokens"])
    line = {"metric": "dispatch+combine tokens/s (gating softmax/top-k + plan + pack + combine; "
                      "router projection and FFN excluded)",
            "value": ref["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1, "steps": None,
            "warmup": 3, "ms_per_step": ref["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg["name"], "experts": E, "top_k": k, "d_model": d,
                       "tokens_per_gpu": cfg["tokens"]},
            "roofline": {"kernel": "lz pack / combine", "bound": "hbm",
                         "achieved": ref["pack_GBps"], "peak": hbm, "unit": "GB/s",
                         "frac": ref["pack_frac"], "combine_frac": ref["combine_frac"],
                         "peak_kind": f"{src} copy bandwidth", "traffic": None},
            "sweep": sweep}
    emit(line)
    return 0


def run_elastic(args, cfg):
    """Config 5: measure the layer on N ranks, remove ranks twice (8 -> 6 -> 4 on 8 GPUs,
    4 -> 3 -> 2 on 4), re-plan on the host with the reference recipe, migrate expert state
    over NVLink, and measure again on the survivors with the SAME kernels.  Slots per GPU
    stay at the full-size value (slots are per-GPU memory)."""
    import torch.distributed as dist

    from paper_2407_04656_b200 import ops
    from paper_2407_04656_b200.elastic import shrink_and_replan
    from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix

    rank, world, local = _env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    E, k, d, dff, Tn = cfg["E"], cfg["k"], cfg["d"], cfg["dff"], cfg["tokens"]
    # slots per GPU held at the 8-GPU value whatever the starting N (slots are per-GPU
    # memory)
    c = math.ceil(cfg["slot_factor"] * E / 8)
    bias = zipf_router_bias(E, cfg["s"], seed=0)
    layer = MoELayer(d, dff, E, k, seed=0, router_bias=bias, device=dev,
                     router_std=1.28 / math.sqrt(d), group=dist.group.WORLD)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn(Tn, d, generator=g, device=dev).bfloat16()
    dout = (torch.randn(Tn, d, generator=g, device=dev) * 1e-2).bfloat16()
    hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3].long()
    dist.all_reduce(hist)
    loads = hist.cpu().tolist()
    layer.set_plan(replica_matrix(plan_for_loads(loads, world, c, 2)))
    group = dist.group.WORLD

    from paper_2407_04656_b200.layer import run_step

    def one_step():
        layer.zero_grad(set_to_none=True)
        layer(x).backward(dout)

    def measure(grp):
        # the first warm-up step applies the capacity protocol: a plan that needs more
        # exchange rows (the survivors' plans are less balanced) grows the buffers before
        # anything is timed; a step that overflowed exchanges nothing and must not be timed
        run_step([layer], one_step)
        for _ in range(max(args.warmup, 3) - 1):
            one_step()
        torch.cuda.synchronize()
        layer.check()
        dist.barrier(group=grp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            layer.zero_grad(set_to_none=True)
            layer(x).backward(dout)
        e1.record()
        torch.cuda.synchronize()
        layer.check()     # every timed step ran the full exchange
        t = torch.tensor([e0.elapsed_time(e1)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=grp)
        n = dist.get_world_size(grp)
        ms = float(t.item()) / args.steps
        return {"n_gpus": n, "ms_per_step": ms, "tokens_per_s": n * Tn / (ms * 1e-3),
                "tokens_per_s_per_gpu": Tn / (ms * 1e-3), "imbalance": round(layer.imbalance(), 4)}

    phases = [measure(group)]
    # two failure events; never remove rank 0 (it reports)
    drops = ([3, 6], [1, 4]) if world == 8 else ([world - 1], [world - 2]) if world >= 4 else ()
    reconf = []
    for ex in drops:
        if dist.get_rank(group) in ex:
            os._exit(0)  # this rank "fails"
        t0 = time.perf_counter()
        layer, group, rep = shrink_and_replan(layer, group, ex, loads, c)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        reconf.append({"excluded": ex, "seconds": round(dt, 3), "transfers": rep["transfers"],
                       "bytes": rep["bytes"], "checkpoint_fallback": len(rep["checkpoint_fallback"]),
                       "replicas": rep["replicas"]})
        phases.append(measure(group))
    if dist.get_rank(group) == 0:
        base = phases[0]["tokens_per_s_per_gpu"]
        for ph in phases:
            ph["retained_per_gpu_vs_full"] = round(ph["tokens_per_s_per_gpu"] / base, 4)
        last = phases[-1]
        line = {"metric": METRIC + " on survivors after elastic reconfiguration",
                "value": last["tokens_per_s"], "unit": "tokens/s", "n_gpus": last["n_gpus"],
                "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": last["ms_per_step"], "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": cfg["name"], "slots_per_gpu": c, "start_gpus": world,
                           "sequence": "->".join(str(p["n_gpus"]) for p in phases)},
                "phases": phases, "reconfigurations": reconf}
        emit(line)
    dist.barrier(group=group)
    dist.destroy_process_group()
    return 0


def plan_replicas(plan, E):
    counts = [0] * E
    for row in plan.slots:
        for v in row:
            counts[v] += 1
    return counts


_OUT = None


def emit(line: dict) -> None:
    """The one JSON line on the real stdout (libraries' own chatter goes to stderr)."""
    out = _OUT if _OUT is not None else sys.stdout
    print(json.dumps(line), file=out, flush=True)


def main():
    global _OUT
    # fd 1 -> stderr for everything else in the process (e.g. NCCL's version banner when
    # NCCL_DEBUG is set on the box), so stdout carries exactly the JSON line
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="lz", choices=["lz", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-isolated", action="store_true",
                    help="skip the isolated per-kernel HBM pass (hbm_kernels)")
    ap.add_argument("--no-graph", action="store_true", help="time eager steps only")
    ap.add_argument("--cpu-reps", type=int, default=12)
    ap.add_argument("--slot-factor", type=float, default=None,
                    help="slots per GPU = ceil(f * E / N) (default: the config's)")
    ap.add_argument("--zipf", type=float, default=None,
                    help="Zipf exponent of the synthetic routing (default: the config's; "
                         "2.5 = the paper-skew variant, top-2 share ~88 %% at E = 16)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.zipf is not None:
        cfg["s"] = args.zipf
    if args.slot_factor is not None:
        cfg["slot_factor"] = args.slot_factor
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.config == "cfg4":
        return run_dispatch_sweep(args, cfg)
    if args.config == "cfg5":
        return run_elastic(args, cfg)
    if args.config == "cfg1" and args.gpus == 1:
        return run_virtual(args, cfg)
    return run_gpu(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
