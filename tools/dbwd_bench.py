"""dispatch-backward / combine-backward kernel timing at cfg2 size (L2 flushed between
reps).  LZ_LIB_PATH selects the liblz build:  python tools/dbwd_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import _lib, ops  # noqa: E402

Tn, d, E, k = 65536, 1024, 16, 2
P = Tn * k
g = torch.Generator(device="cuda").manual_seed(0)
rows = torch.randperm(P, device="cuda", generator=g).int().view(Tn, k)
dxe = torch.randn(P, d, device="cuda", generator=g).bfloat16()
logits = torch.randn(Tn, E, device="cuda", generator=g)
probs = torch.softmax(logits, 1)
idx = torch.topk(logits, k, 1).indices.int()
dw = torch.randn(Tn, k, device="cuda", generator=g)
wg = (torch.randn(E, d, device="cuda", generator=g) * 0.04).bfloat16()
w = torch.rand(Tn, k, device="cuda", generator=g)
dout = torch.randn(Tn, d, device="cuda", generator=g).bfloat16()
y = torch.randn(P, d, device="cuda", generator=g).bfloat16()
dy = torch.empty_like(y)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, name, nbytes):
    ts = []
    for i in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"{os.environ.get('LZ_LIB_PATH', 'liblz.so')}: {name} min {ts[0]:.1f} us "
          f"({nbytes / (ts[0] * 1e-6) / 1e12:.2f} TB/s)")


t(lambda: ops.dispatch_bwd(dxe, rows.view(-1), probs, idx, dw, wg, False, Tn), "dispatch_bwd",
  P * d * 2 + Tn * d * 2 + 2 * Tn * E * 4)
t(lambda: ops.combine_bwd(dout, y, rows.view(-1), w, k, dy), "combine_bwd",
  Tn * d * 2 + 2 * P * d * 2 + P * 8)
t(lambda: ops.dispatch_bwd(dxe, rows.view(-1), probs, idx, dw, None, False, Tn),
  "dispatch_bwd (no router term)", P * d * 2 + Tn * d * 2 + 2 * Tn * E * 4)
seq_rows = torch.arange(P, dtype=torch.int32, device="cuda")
t(lambda: ops.dispatch_bwd(dxe, seq_rows, probs, idx, dw, None, False, Tn),
  "dispatch_bwd (no router term, sequential rows)", P * d * 2 + Tn * d * 2 + 2 * Tn * E * 4)
t(lambda: ops.combine_bwd(dout, y, seq_rows, w, k, dy), "combine_bwd (sequential rows)",
  Tn * d * 2 + 2 * P * d * 2 + P * 8)
t(lambda: ops.router_wgrad(logits, dout), "router_wgrad", Tn * d * 2 + Tn * E * 4)
