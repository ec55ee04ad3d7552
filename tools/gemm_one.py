"""Run lz grouped GEMMs of the cfg2 / cfg3 step shapes (Zipf(1.2) group sizes, as
tools/vendor_bar.py), each ``--reps`` times, for ncu captures:

    ncu --set full -k regex:grouped_gemm -s <warm> -c <n> python tools/gemm_one.py --shape cfg3 \
        --kinds wgrad2,dgrad2 --reps 2

Kinds: fwd1 (store), fwd1_act (GELU / SwiGLU epilogue), fwd2, dgrad1_dact, dgrad2, wgrad1,
wgrad2.  Launch order: kinds in the given order, reps each."""

from __future__ import annotations

import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2407_04656_b200 import _lib, ops  # noqa: E402
from vendor_bar import group_sizes, timeit  # noqa: E402

SHAPES = {"cfg2": (16, 2, 65536, 1024, 4096, False), "cfg3": (8, 2, 16384, 4096, 14336, True)}


def build(shape):
    E, k, T, d, dff, swi = SHAPES[shape]
    dev = torch.device("cuda")
    m = group_sizes(E, k, T, 1.2)
    align = ops.row_align()
    mp = [(v + align - 1) // align * align for v in m]
    rows = sum(mp)
    off = torch.tensor([0] + list(torch.tensor(mp).cumsum(0)), dtype=torch.int32, device=dev)
    f1 = 2 * dff if swi else dff
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    X = torch.randn(rows, d, generator=g, device=dev).bfloat16()
    W1 = (torch.randn(E, f1, d, generator=g, device=dev) * 0.02).bfloat16()
    W2 = (torch.randn(E, d, dff, generator=g, device=dev) * 0.02).bfloat16()
    H = torch.empty(rows, f1, dtype=torch.bfloat16, device=dev)
    A = torch.randn(rows, dff, generator=g, device=dev).bfloat16()
    Y = torch.empty(rows, d, dtype=torch.bfloat16, device=dev)
    dY = torch.randn(rows, d, generator=g, device=dev).bfloat16()
    dH = torch.empty(rows, f1, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(rows, d, dtype=torch.bfloat16, device=dev)
    dW1, dW2 = torch.empty_like(W1), torch.empty_like(W2)
    act, dact = ((_lib.LZ_EPI_SWIGLU, _lib.LZ_EPI_DSWIGLU) if swi
                 else (_lib.LZ_EPI_GELU, _lib.LZ_EPI_DGELU))
    MN = _lib.LZ_MN_MAJOR
    kinds = {
        "fwd1": lambda: ops.grouped_gemm_rows(X, W1, off, H),
        "fwd1_act": lambda: ops.grouped_gemm_rows(X, W1, off, A, aux=H, epilogue=act),
        "fwd2": lambda: ops.grouped_gemm_rows(A, W2, off, Y),
        "dgrad1_dact": lambda: ops.grouped_gemm_rows(dY, W2, off, dH, b_major=MN, aux=H,
                                                     epilogue=dact),
        "dgrad2": lambda: ops.grouped_gemm_rows(dH, W1, off, dX, b_major=MN),
        "wgrad1": lambda: ops.grouped_gemm_wgrad(dH, X, off, dW1),
        "wgrad2": lambda: ops.grouped_gemm_wgrad(dY, A, off, dW2),
    }
    flops = {kk: 2.0 * sum(m) * d * dff * (2 if swi and kk in ("fwd1", "fwd1_act", "dgrad2",
                                                               "wgrad1") else 1)
             for kk in kinds}
    return kinds, flops


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="cfg2", choices=sorted(SHAPES))
    ap.add_argument("--kinds", default="fwd1_act,fwd2,dgrad1_dact,dgrad2,wgrad1,wgrad2")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--time", action="store_true", help="print CUDA-event times instead")
    a = ap.parse_args()
    _lib.load()
    kinds, flops = build(a.shape)
    for name in a.kinds.split(","):
        if a.time:
            ms = timeit(kinds[name])
            print(f"{a.shape} {name:12s} {ms * 1e3:8.1f} us {flops[name] / ms / 1e9:7.1f} TFLOP/s",
                  flush=True)
        else:
            for _ in range(a.reps):
                kinds[name]()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
