"""Diagnostic: cluster GEMM in eager launches vs CUDA-graph replay (not collected)."""
import os, sys, time, subprocess
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops

torch.manual_seed(0)
rows, K, N, G = 131072 + 4096, 1024, 4096, 16
seg = [8192 + 256] * 16
off = torch.tensor([0] + list(torch.tensor(seg).cumsum(0)), dtype=torch.int32, device="cuda")
A = torch.randn(rows, K, device="cuda").bfloat16()
B = torch.randn(G, N, K, device="cuda").bfloat16() * 0.03
C = torch.empty(rows, N, device="cuda").bfloat16()
H = torch.empty(rows, N, device="cuda").bfloat16()

def launches(n, epi):
    for _ in range(n):
        ops.grouped_gemm_rows(A, B, off, C, epilogue=epi, aux=H if epi else None)

for epi, direct in ((0, 0), (0, 1), (1, 0), (1, 1)):
    for cg in (2,):
        ops.set_gemm_cta_group(cg)
        ops.set_gemm_direct_epilogue(direct)
        launches(3, epi); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); launches(20, epi); e1.record(); torch.cuda.synchronize()
        t_eager = e0.elapsed_time(e1) / 20
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            launches(1, epi)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            launches(20, epi)
        g.replay(); torch.cuda.synchronize()
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        t_graph = e0.elapsed_time(e1) / 20
        fl = 2 * (rows - 4096) * K * N
        print(f"epi={epi} direct={direct} cg={cg}: eager {t_eager:.3f} ms ({fl / t_eager / 1e9:.0f} TF/s)  graph {t_graph:.3f} ms ({fl / t_graph / 1e9:.0f} TF/s)", flush=True)

# dgrad-like: MN-major B with DGELU epilogue
Bm = torch.randn(G, K, N, device="cuda").bfloat16() * 0.03
for direct in (0, 1, 2):
    ops.set_gemm_direct_epilogue(direct)
    f = lambda: ops.grouped_gemm_rows(A, Bm, off, C, b_major=1, epilogue=2, aux=H)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        f()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    print(f"dgelu direct={direct}: {t:.3f} ms ({2 * (rows - 4096) * K * N / t / 1e9:.0f} TF/s)", flush=True)
