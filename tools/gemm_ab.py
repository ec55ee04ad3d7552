"""Interleaved A/B of the grouped GEMM between two liblz builds in ONE process.

    python tools/gemm_ab.py build/ab/liblz_base.so paper_2407_04656_b200/liblz.so [--swiglu]

Each trial runs a short burst (3 launches) of one GEMM from lib A, sleeps, then the same
from lib B, so both see the same power/thermal state (B200 runs at its power cap under
sustained tensor load; back-to-back loops drift by +-10 %).  Reports min and median
per-launch time over the trials."""

from __future__ import annotations

import argparse
import ctypes
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2407_04656_b200 import _lib  # noqa: E402


def load(path):
    h = ctypes.CDLL(os.path.abspath(path))
    h.lz_grouped_gemm.argtypes = _lib._SIGS["lz_grouped_gemm"]
    h.lz_grouped_gemm.restype = ctypes.c_int
    return h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib_a")
    ap.add_argument("lib_b")
    ap.add_argument("--swiglu", action="store_true")
    ap.add_argument("--trials", type=int, default=15)
    ap.add_argument("--groups", type=int, default=16)
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--dff", type=int, default=4096)
    ap.add_argument("--rows", type=int, default=131072)
    a = ap.parse_args()
    libs = [load(a.lib_a), load(a.lib_b)]
    G, d, dff = a.groups, a.d, a.dff
    torch.manual_seed(0)
    # Zipf(1.2)-like group sizes (the cfg2 routing), 256-row padded
    w = torch.tensor([(1 + e) ** -1.2 for e in range(G)])
    m = [int(v) // 256 * 256 + 256 for v in (w / w.sum() * a.rows)]
    off = torch.tensor([0] + torch.tensor(m).cumsum(0).tolist(), dtype=torch.int32, device="cuda")
    rows = int(off[-1])
    f1 = 2 * dff if a.swiglu else dff
    bf = dict(device="cuda", dtype=torch.bfloat16)
    X = torch.randn(rows, d, **bf)
    W1 = torch.randn(G, f1, d, **bf) * 0.02
    W2 = torch.randn(G, d, dff, **bf) * 0.02
    H = torch.empty(rows, f1, **bf)
    A = torch.empty(rows, dff, **bf)
    Y = torch.empty(rows, d, **bf)
    dY = torch.randn(rows, d, **bf)
    dA = torch.empty(rows, f1, **bf)
    dX = torch.empty(rows, d, **bf)
    dW1 = torch.empty_like(W1)
    dW2 = torch.empty_like(W2)
    act, dact = ((_lib.LZ_EPI_SWIGLU, _lib.LZ_EPI_DSWIGLU) if a.swiglu
                 else (_lib.LZ_EPI_GELU, _lib.LZ_EPI_DGELU))
    p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    s = torch.cuda.current_stream().cuda_stream
    K, MN = _lib.LZ_K_MAJOR, _lib.LZ_MN_MAJOR
    # name: (mode, A, B, C, aux, M, N, K, b_major, epilogue)
    cases = {
        "fwd1 store": (0, X, W1, H, None, 0, f1, d, K, _lib.LZ_EPI_STORE),
        "fwd1+act": (0, X, W1, A, H, 0, f1, d, K, act),
        "fwd2": (0, A, W2, Y, None, 0, d, dff, K, _lib.LZ_EPI_STORE),
        "dgrad2+dact": (0, dY, W2, dA, H, 0, dff, d, MN, dact),
        "wgrad2": (1, dY, A, dW2, None, d, dff, 0, MN, _lib.LZ_EPI_STORE),
        "wgrad1": (1, dA, X, dW1, None, f1, d, 0, MN, _lib.LZ_EPI_STORE),
        "dgrad1": (0, dA, W1, dX, None, 0, d, f1, MN, _lib.LZ_EPI_STORE),
    }
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    tot = [0.0, 0.0]
    for name, (mode, Ain, B, C, aux, M, N, Kd, bm, epi) in cases.items():
        def run(h):
            st = h.lz_grouped_gemm(mode, p(Ain), p(B), p(C), p(aux), G, p(off), rows, M, N, Kd,
                                   bm, epi, 0, 0, 0, s)
            assert st == 0, st
        for h in libs:
            run(h)
        torch.cuda.synchronize()
        res = [[], []]
        for _ in range(a.trials):
            for i, h in enumerate(libs):
                time.sleep(0.05)
                ev[0].record()
                for _ in range(3):
                    run(h)
                ev[1].record()
                torch.cuda.synchronize()
                res[i].append(ev[0].elapsed_time(ev[1]) / 3 * 1e3)
        line = []
        for i in range(2):
            tot[i] += min(res[i])
            line.append(f"min {min(res[i]):7.1f} med {statistics.median(res[i]):7.1f}")
        print(f"{name:12s} A: {line[0]}   B: {line[1]}   B/A(min) {min(res[1]) / min(res[0]):.3f}",
              flush=True)
    print(f"total(min)   A {tot[0]:.1f} us   B {tot[1]:.1f} us   B/A {tot[1] / tot[0]:.3f}")
    # library reference: the same per-expert products through cuBLAS (torch.mm per group,
    # bf16 in/out, fp32 accumulate) -- what a library-only grouped GEMM would achieve
    bounds = off.tolist()
    refs = {
        "fwd2": lambda: [torch.mm(A[bounds[g]:bounds[g + 1]], W2[g].t(),
                                  out=Y[bounds[g]:bounds[g + 1]]) for g in range(G)],
        "wgrad2": lambda: [torch.mm(dY[bounds[g]:bounds[g + 1]].t(), A[bounds[g]:bounds[g + 1]],
                                    out=dW2[g]) for g in range(G)],
        "dense fwd2": lambda: torch.mm(A, W2[0].t(), out=Y),
    }
    for name, fn in refs.items():
        fn()
        torch.cuda.synchronize()
        res = []
        for _ in range(a.trials):
            time.sleep(0.05)
            ev[0].record()
            for _ in range(3):
                fn()
            ev[1].record()
            torch.cuda.synchronize()
            res.append(ev[0].elapsed_time(ev[1]) / 3 * 1e3)
        print(f"cuBLAS {name:12s} min {min(res):7.1f} med {statistics.median(res):7.1f} us", flush=True)


if __name__ == "__main__":
    main()
