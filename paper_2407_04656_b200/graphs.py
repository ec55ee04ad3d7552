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
    def __init__(self, layer, tokens: int, nbuf: int = 2, warmup: int = 3, backward: bool = True):
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
        from . import _lib
        for i in range(nbuf):
            layer.zero_grad(set_to_none=True)
            g = torch.cuda.CUDAGraph()
            l0 = _lib.launch_count
            # thread_local: other threads (the NCCL watchdog polling its events) keep
            # running while this thread captures
            with torch.cuda.graph(g, pool=pool, capture_error_mode="thread_local"):
                out = layer(self.x[i])
                if backward:
                    out.backward(self.dout[i])
                # the step's scalar result (checksum of the layer output), read back by e2e
                self.result[i] = out.detach().sum(dtype=torch.float32).view(1)
            self.launches_per_step = _lib.launch_count - l0
            pool = g.pool()
            self.graphs.append(g)
            self.grads.append([p.grad for p in params])
            del out
        self.params = params

    def replay(self, i: int = 0) -> torch.Tensor:
        self.graphs[i].replay()
        for p, gr in zip(self.params, self.grads[i]):
            p.grad = gr
        return self.result[i]
