import os, sys, torch
sys.path.insert(0, "/root/repo") if os.path.isdir("/root/repo") else None
sys.path.insert(0, os.getcwd())
from paper_2407_04656_b200 import ops, _lib
Tn, d, E = 65536, 1024, 16
x = torch.randn(Tn, d, device="cuda").bfloat16()
dl = torch.randn(Tn, E, device="cuda")
xs = [x, x.clone()]
fn = lambda i: ops.router_wgrad(dl, xs[i])
for i in range(4): fn(i & 1)
torch.cuda.synchronize()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(20): fn(i & 1)
g.replay(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); g.replay(); b.record(); torch.cuda.synchronize()
us = a.elapsed_time(b) / 20 * 1e3
ref = (dl.t() @ x.float())
got = ops.router_wgrad(dl, x)[0]
print(os.environ.get("LZ_LIB_PATH"), f"{us:.1f} us", f"{138.4e6/(us*1e-6)/1e9/6544:.3f}", float((got-ref).abs().max()/ref.abs().max()))
