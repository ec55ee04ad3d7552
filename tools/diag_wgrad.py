"""Diagnostic: wgrad GEMM at layer-like shapes for both variants (not collected)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops
torch.manual_seed(0)
for cg in (1, 2):
    ops.set_gemm_cta_group(cg)
    for sizes, M, N, cap in (([256, 512, 0, 256, 768, 256, 256, 512], 2048, 512, 4096),
                             ([256, 512, 0, 256], 256, 512, 1024), ([256] * 8, 1024, 256, 2048)):
        off = torch.tensor([0] + list(torch.tensor(sizes).cumsum(0)), dtype=torch.int32, device="cuda")
        A = torch.randn(cap, M, device="cuda").bfloat16()
        B = torch.randn(cap, N, device="cuda").bfloat16()
        C = torch.full((len(sizes), M, N), float("nan"), device="cuda").bfloat16()
        ops.grouped_gemm_wgrad(A, B, off, C)
        torch.cuda.synchronize()
        worst = 0.0
        o = off.tolist()
        for g in range(len(sizes)):
            ref = A[o[g]:o[g + 1]].float().t() @ B[o[g]:o[g + 1]].float()
            err = ((C[g].float() - ref).norm() / ref.norm().clamp_min(1e-9)).item() if o[g + 1] > o[g] \
                else C[g].float().abs().max().item()
            worst = max(worst, err)
        print(f"cg={cg} sizes={sizes} M={M} N={N}: worst rel err {worst:.3e}", flush=True)
