"""Host -> device input pipeline for the layer's public API (pinned memory, side stream).

``HostPrefetcher(host_tensors, device)``: ``prefetch()`` starts non-blocking H2D copies of
the pinned host tensors on a dedicated copy stream; ``get()`` makes the current stream
wait for them and returns the device tensors (recorded on the consumer stream so the
caching allocator never recycles them early).  Double buffering lets the copy of step
i+1 overlap the compute of step i over PCIe while every byte still crosses per step.
"""

from __future__ import annotations

import collections

import torch


class HostPrefetcher:
    def __init__(self, host_tensors, device):
        self.host = list(host_tensors)
        self.device = device
        self.stream = torch.cuda.Stream(device=device)
        self.pending = collections.deque()

    def prefetch(self) -> None:
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            dev = [t.to(self.device, non_blocking=True) for t in self.host]
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.pending.append((dev, ev))

    def get(self):
        dev, ev = self.pending.popleft()
        cur = torch.cuda.current_stream(self.device)
        cur.wait_event(ev)
        for t in dev:
            t.record_stream(cur)
        return dev
