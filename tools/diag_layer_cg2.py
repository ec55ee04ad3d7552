"""Diagnostic: layer gradients for cg=1 vs cg=2 and GEMM determinism (not collected)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix

res = {}
for cg in (1, 2):
    ops.set_gemm_cta_group(cg)
    torch.manual_seed(0)
    for (Tn, d, dff, E, k, s) in [(1024, 512, 2048, 8, 2, 1.2), (2048, 1024, 4096, 16, 2, 2.5)]:
        layer = MoELayer(d, dff, E, k, seed=3, init_std=0.05, router_bias=zipf_router_bias(E, s, seed=1))
        layer.set_plan(replica_matrix(plan_for_loads([100 * (e + 1) for e in range(E)], 1, 3 * E)))
        x = torch.randn(Tn, d, device="cuda").bfloat16().requires_grad_(True)
        out = layer(x)
        dout = torch.randn_like(out)
        out.backward(dout)
        torch.cuda.synchronize()
        res[(cg, Tn)] = (out.float().cpu(), x.grad.float().cpu(), layer.w1.grad.float().cpu(),
                         layer.w2.grad.float().cpu(), layer.last_plan.recv_off.cpu(), layer.local_ids)
for Tn in (1024, 2048):
    a, b = res[(1, Tn)], res[(2, Tn)]
    print("Tn", Tn, "off cg1", a[4].tolist()[:6], "cg2", b[4].tolist()[:6])
    for name, u, v in zip(["out", "dx", "dW1", "dW2"], a[:4], b[:4]):
        if u.shape != v.shape:
            print(name, "shape", u.shape, v.shape); continue
        e = ((u - v).norm() / u.norm()).item()
        print(f"  {name}: rel diff cg1 vs cg2 {e:.3e}")
        if name in ("dW1", "dW2"):
            for g in range(u.shape[0]):
                eg = ((u[g] - v[g]).norm() / u[g].norm().clamp_min(1e-9)).item()
                if eg > 1e-2:
                    print(f"     group {g} expert {a[5][g]} rel diff {eg:.3e} norm1 {u[g].norm():.3e} norm2 {v[g].norm():.3e}")
