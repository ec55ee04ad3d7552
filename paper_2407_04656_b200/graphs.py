"""CUDA-graph capture of a whole MoE-layer training step (forward + backward).

At N = 1 and with the fused P2P exchange at N > 1 the step has no host
synchronisation, so it is captured once and replayed: one graph launch per step
instead of ~20 library calls and ~40 torch allocations, and the step becomes immune
to host jitter.  ``nbuf`` static input slots (x, upstream gradient) let the caller
stream inputs in from the host while another slot's replay runs (double buffering).

Replays overwrite the parameter gradients (captured with ``.grad`` unset), exactly
what a fresh ``zero_grad(set_to_none=True)`` + forward + backward produces.
"""

from __future__ import annotations

import torch


class GraphedStep:
    def __init__(self, layer, tokens: int, nbuf: int = 2, warmup: int = 3, backward: bool = True,
                 timed_slot: int | None = None):
        """timed_slot: that slot's graph also records CUDA events (graph event-record
        nodes) around the whole step and around every grouped-GEMM launch, so each of its
        replays is timed from inside the graph (``replay_times``)."""
        dev = layer.device
        d = layer.d
        self.layer = layer
        self.x = [torch.zeros(tokens, d, dtype=torch.bfloat16, device=dev) for _ in range(nbuf)]
        self.dout = [torch.zeros(tokens, d, dtype=torch.bfloat16, device=dev) for _ in range(nbuf)]
        self.result = [None] * nbuf
        self.graphs = []
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                layer.zero_grad(set_to_none=True)
                out = layer(self.x[0])
                if backward:
                    out.backward(self.dout[0])
                del out  # no autograd node (AccumulateGrad) may outlive the iteration
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        # blocks freed with pending cross-stream uses (record_stream) are reclaimed by
        # querying events -- illegal inside a capture; settle them now
        torch.cuda.empty_cache()
        pool = None
        self.grads = []
        params = [p for p in layer.parameters() if p.requires_grad]
        from . import _lib, ops
        self.step_events = None
        self.gemm_events = None
        for i in range(nbuf):
            layer.zero_grad(set_to_none=True)
            g = torch.cuda.CUDAGraph()
            l0 = _lib.launch_count
            timed = i == timed_slot
            if timed:
                ops.GEMM_EVENTS, ops.GEMM_EVENTS_EXTERNAL = [], True
                self.step_events = (torch.cuda.Event(enable_timing=True, external=True),
                                    torch.cuda.Event(enable_timing=True, external=True))
            # thread_local: other threads (the NCCL watchdog polling its events) keep
            # running while this thread captures
            try:
                with torch.cuda.graph(g, pool=pool, capture_error_mode="thread_local"):
                    if timed:
                        self.step_events[0].record()
                    out = layer(self.x[i])
                    if backward:
                        out.backward(self.dout[i])
                    # the step's scalar result (checksum of the layer output), read by e2e
                    self.result[i] = out.detach().sum(dtype=torch.float32).view(1)
                    if timed:
                        self.step_events[1].record()
            finally:
                if timed:
                    self.gemm_events = ops.GEMM_EVENTS
                    ops.GEMM_EVENTS, ops.GEMM_EVENTS_EXTERNAL = None, False
            if i == 0:
                self.launches_per_step = _lib.launch_count - l0
            pool = g.pool()
            self.graphs.append(g)
            self.grads.append([p.grad for p in params])
            del out
        self.params = params
        self._timed = timed_slot

    def replay(self, i: int = 0) -> torch.Tensor:
        self.graphs[i].replay()
        for p, gr in zip(self.params, self.grads[i]):
            p.grad = gr
        return self.result[i]

    def replay_times(self, n: int) -> dict:
        """Replay the timed slot n times (synchronising after each, so its in-graph events
        can be read) -> per-replay step and grouped-GEMM milliseconds measured by the
        graph's own event nodes, i.e. within the same replays."""
        if self.step_events is None:
            raise RuntimeError("no timed slot captured")
        slot = self._timed
        steps, gemms, per_launch = [], [], []
        for _ in range(n):
            self.replay(slot)
            torch.cuda.synchronize()
            steps.append(self.step_events[0].elapsed_time(self.step_events[1]))
            ts = [a.elapsed_time(b) for a, b in self.gemm_events]
            gemms.append(sum(ts))
            per_launch.append(ts)
        return {"step_ms": steps, "gemm_ms": gemms, "gemm_launch_ms": per_launch}
