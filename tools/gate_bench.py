"""Router-gate kernel timing across liblz builds: python tools/gate_bench.py lib1.so lib2.so ..."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_04656_b200 import _lib  # noqa: E402

Tn, d, E, k = (int(v) for v in os.environ.get("GATE_SHAPE", "65536,1024,16,2").split(","))
x = torch.randn(Tn, d, device="cuda").bfloat16()
wg = (torch.randn(E, d, device="cuda") * 0.04).bfloat16()
bg = torch.zeros(E, device="cuda")
idx = torch.empty(Tn, k, dtype=torch.int32, device="cuda")
w = torch.empty(Tn, k, device="cuda")
probs = torch.empty(Tn, E, device="cuda")
hist = torch.empty(E, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for path in sys.argv[1:]:
    h = ctypes.CDLL(os.path.abspath(path))
    h.lz_router_gate.argtypes = _lib._SIGS["lz_router_gate"]
    ts = []
    for i in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st = h.lz_router_gate(x.data_ptr(), wg.data_ptr(), bg.data_ptr(), Tn, d, E, k, 0,
                              idx.data_ptr(), w.data_ptr(), probs.data_ptr(), hist.data_ptr(), s)
        b.record()
        torch.cuda.synchronize()
        assert st == 0
        if i >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    nbytes = Tn * d * 2
    print(f"{path} [{Tn}x{d}, E{E} k{k}]: min {ts[0]:.1f} med {ts[len(ts)//2]:.1f} us  "
          f"({nbytes / (ts[0] * 1e-6) / 1e12:.2f} TB/s)")
