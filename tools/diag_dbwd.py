"""Diagnostic: dispatch_bwd / combine_bwd / combine kernel timings in isolation."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import ops
torch.manual_seed(0)
Tn, d, E, k = 65536, 1024, 16, 2
P = Tn * k
rows = torch.randperm(P + 4096, device="cuda")[:P].int()
dxe = torch.randn(P + 4096, d, device="cuda").bfloat16()
probs = torch.softmax(torch.randn(Tn, E, device="cuda"), 1)
idx = torch.topk(probs, k, 1).indices.int()
dw = torch.randn(Tn, k, device="cuda")
wg = (torch.randn(E, d, device="cuda") * 0.03).bfloat16()
w = torch.rand(Tn, k, device="cuda")
x = torch.randn(Tn, d, device="cuda").bfloat16()
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000
seq = torch.arange(P, device="cuda").int()
print("dispatch_bwd full       %.1f us" % t(lambda: ops.dispatch_bwd(dxe, rows, probs, idx, dw, wg, False, Tn)))
print("dispatch_bwd sequential %.1f us" % t(lambda: ops.dispatch_bwd(dxe, seq, probs, idx, dw, wg, False, Tn)))
print("dispatch_bwd no router  %.1f us" % t(lambda: ops.dispatch_bwd(dxe, rows, probs, idx, dw, None if False else wg[:0].view(0, d) if False else wg, False, Tn)))
dy = torch.empty_like(dxe)
print("combine_bwd             %.1f us" % t(lambda: ops.combine_bwd(x, dxe, rows, w, k, dy)))
print("combine                 %.1f us" % t(lambda: ops.combine(dxe, rows, w, k)))
dl = torch.randn(Tn, E, device="cuda")
print("router_wgrad            %.1f us" % t(lambda: ops.router_wgrad(dl, x)))
print("router_gate             %.1f us" % t(lambda: ops.router_gate(x, wg, None, k)))
print("bytes: dispatch_bwd alg %.0f MB" % ((P * d * 2 + Tn * d * 2 + Tn * E * 8) / 1e6))
