"""Diagnostic: which liblz call breaks CUDA-graph capture (not collected)."""
import os, sys, traceback
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops
from paper_2407_04656_b200.dispatch import plan_device

dev = torch.device("cuda", 0)
E, k, d, Tn = 16, 2, 1024, 4096
x = torch.randn(Tn, d, device=dev).bfloat16()
wg = torch.randn(E, d, device=dev).bfloat16() * 0.02
bg = torch.zeros(E, device=dev)
R = torch.ones(E, 1, dtype=torch.int32, device=dev)

def try_capture(name, fn):
    fn()  # warm
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        print(f"{name}: OK", flush=True)
    except Exception as e:
        print(f"{name}: FAIL {repr(e)[:150]}", flush=True)
        torch.cuda.synchronize()

try_capture("router_gate", lambda: ops.router_gate(x, wg, bg, k))
idx, w, probs, hist = ops.router_gate(x, wg, bg, k)
try_capture("plan_device", lambda: plan_device(hist.view(E, 1), R, 0, idx.view(-1), 256))
p = plan_device(hist.view(E, 1), R, 0, idx.view(-1), 256)
X = torch.empty(Tn * k + E * 256, d, device=dev).bfloat16()
try_capture("pack", lambda: ops.pack(x, p.dest_row, k, X, p.recv_m, p.recv_off))
try_capture("combine", lambda: ops.combine(X, p.dest_row, w, k))
W = torch.randn(E, 256 * 4, d, device=dev).bfloat16()
Hb = torch.empty(X.shape[0], 1024, device=dev).bfloat16()
try_capture("gemm", lambda: ops.grouped_gemm_rows(X, W, p.recv_off, Hb))

from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
layer = MoELayer(d, 4096, E, k, router_bias=zipf_router_bias(E, 1.2), device=dev)
xx = torch.randn(Tn, d, device=dev).bfloat16()
dd = torch.randn(Tn, d, device=dev).bfloat16()
try_capture("layer fwd (no grad)", lambda: layer(xx.detach()) if torch.no_grad().__enter__() is None else None)
torch.set_grad_enabled(True)
def fwdbwd():
    out = layer(xx)
    out.backward(dd)
for mode in ("global", "thread_local", "relaxed"):
    fwdbwd(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, capture_error_mode=mode):
            fwdbwd()
        g.replay(); torch.cuda.synchronize()
        print(f"layer fwd+bwd capture mode {mode}: OK", flush=True)
    except Exception as e:
        print(f"layer fwd+bwd capture mode {mode}: FAIL {repr(e)[:300]}", flush=True)
        try:
            torch.cuda.synchronize()
        except Exception as e2:
            print("  sync:", repr(e2)[:100])
