"""Power-settled GEMM throughput: each candidate runs back-to-back for `--secs` seconds
and the rate over the last third is reported (B200 sits at its power cap under sustained
tensor load, so this is the energy efficiency of the kernel, not its burst speed).

    python tools/gemm_sustained.py [--secs 6]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import _lib, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--secs", type=float, default=6.0)
a = ap.parse_args()
G, d, dff, rows = 16, 1024, 4096, 131072
w = torch.tensor([(1 + e) ** -1.2 for e in range(G)])
m = [int(v) // 256 * 256 + 256 for v in (w / w.sum() * rows)]
off = torch.tensor([0] + torch.tensor(m).cumsum(0).tolist(), dtype=torch.int32, device="cuda")
R = int(off[-1])
bf = dict(device="cuda", dtype=torch.bfloat16)
X = torch.randn(R, d, **bf)
A = torch.randn(R, dff, **bf)
W1 = torch.randn(G, dff, d, **bf) * 0.02
W2 = torch.randn(G, d, dff, **bf) * 0.02
H = torch.empty(R, dff, **bf)
Y = torch.empty(R, d, **bf)
flops = 2.0 * R * d * dff
W0 = W2[0].contiguous()
cands = {
    "ours fwd2 (store epilogue)": lambda: ops.grouped_gemm_rows(A, W2, off, Y),
    "ours fwd1 (GELU, 2 outputs)": lambda: ops.grouped_gemm_rows(X, W1, off, A, aux=H,
                                                                 epilogue=_lib.LZ_EPI_GELU),
    "cuBLAS dense same size": lambda: torch.mm(A, W0.t(), out=Y),
}
for name, fn in cands.items():
    fn()
    torch.cuda.synchronize()
    t_end = time.time() + a.secs
    marks = []
    while time.time() < t_end:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        marks.append(e0.elapsed_time(e1) / 20)
    tail = marks[len(marks) * 2 // 3:]
    ms = sum(tail) / len(tail)
    print(f"{name:30s} first {marks[0]:.3f} ms, settled {ms:.3f} ms = "
          f"{flops / (ms * 1e-3) / 1e12:.0f} TFLOP/s", flush=True)
    time.sleep(3)
