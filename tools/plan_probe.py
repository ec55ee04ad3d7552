"""Planning kernels alone (count / plan / slot) at P routed assignments over E experts:
    python tools/plan_probe.py [P] [E]"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))
from paper_2407_04656_b200.dispatch import plan_device  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
E = int(sys.argv[2]) if len(sys.argv) > 2 else 64
p = torch.tensor([(1 + e) ** -1.5 for e in range(E)])
routed = torch.multinomial(p, P, replacement=True).int().cuda()
hist = torch.bincount(routed.long(), minlength=E).int().view(E, 1).cuda()
R = torch.full((E, 1), 2, dtype=torch.int32, device="cuda")
for _ in range(3):
    plan_device(hist, R, 0, routed, 256)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    plan_device(hist, R, 0, routed, 256)
b.record()
torch.cuda.synchronize()
print(f"plan_device P={P} E={E}: {a.elapsed_time(b) / 20 * 1e3:.1f} us per call")
