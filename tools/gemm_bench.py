"""A/B microbenchmark of the six grouped GEMMs of one cfg2 step (E=16 groups, 131,072
routed rows + 256-row padding, d=1024, d_ff=4096), CUDA-event timed, L2-resident
weights, inputs >> L2.  Usage: python tools/gemm_bench.py [--reps 20] [--swiglu]"""

from __future__ import annotations

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2407_04656_b200 import _lib, ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--swiglu", action="store_true")
    a = ap.parse_args()
    G, d, dff = 16, 1024, 4096
    torch.manual_seed(0)
    sizes = torch.distributions.Dirichlet(torch.ones(G)).sample() * 131072
    m = [int(v) // 256 * 256 + 256 for v in sizes]
    off = torch.tensor([0] + torch.tensor(m).cumsum(0).tolist(), dtype=torch.int32, device="cuda")
    rows = int(off[-1])
    f1 = 2 * dff if a.swiglu else dff
    X = torch.randn(rows, d, device="cuda").bfloat16()
    W1 = (torch.randn(G, f1, d, device="cuda") * 0.02).bfloat16()
    W2 = (torch.randn(G, d, dff, device="cuda") * 0.02).bfloat16()
    H = torch.empty(rows, f1, device="cuda", dtype=torch.bfloat16)
    A = torch.empty(rows, dff, device="cuda", dtype=torch.bfloat16)
    Y = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    dY = torch.randn(rows, d, device="cuda").bfloat16()
    dA = torch.empty(rows, f1, device="cuda", dtype=torch.bfloat16)
    dX = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    dW1 = torch.empty_like(W1)
    dW2 = torch.empty_like(W2)
    act, dact = ((_lib.LZ_EPI_SWIGLU, _lib.LZ_EPI_DSWIGLU) if a.swiglu
                 else (_lib.LZ_EPI_GELU, _lib.LZ_EPI_DGELU))
    ops_ = {
        "fwd1+act": lambda: ops.grouped_gemm_rows(X, W1, off, A, aux=H, epilogue=act),
        "fwd2": lambda: ops.grouped_gemm_rows(A, W2, off, Y),
        "dgrad2+dact": lambda: ops.grouped_gemm_rows(dY, W2, off, dA, b_major=_lib.LZ_MN_MAJOR,
                                                     aux=H, epilogue=dact),
        "wgrad2": lambda: ops.grouped_gemm_wgrad(dY, A, off, dW2),
        "wgrad1": lambda: ops.grouped_gemm_wgrad(dA, X, off, dW1),
        "dgrad1": lambda: ops.grouped_gemm_rows(dA, W1, off, dX, b_major=_lib.LZ_MN_MAJOR),
    }
    n_mat = 3 if a.swiglu else 2
    # fwd1 / wgrad1 / dgrad1 touch W1 (2 d_ff rows for SwiGLU: gate | up)
    flops = {k: 2 * rows * d * dff * (2 if a.swiglu and k in ("fwd1+act", "wgrad1", "dgrad1")
                                      else 1) for k in ops_}
    tot = 0.0
    for name, fn in ops_.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        tot += ms
        print(f"{name:12s} {ms * 1e3:8.1f} us  {flops[name] / ms / 1e9:7.1f} TFLOP/s", flush=True)
    print(f"total        {tot * 1e3:8.1f} us  ({n_mat} matrices)")


if __name__ == "__main__":
    main()
