"""Pinned host -> device copy bandwidth: one stream vs two streams vs chunked (the e2e
input path of bench.py is bound by it).   python tools/h2d_bw.py"""
import torch

n = 128 << 20
xs = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(4)]


def run(mode):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    if mode == "1 stream":
        for i in range(2):
            ds[i].copy_(xs[i], non_blocking=True)
    elif mode == "2 streams":
        for i in range(2):
            streams[i].wait_event(a)
            with torch.cuda.stream(streams[i]):
                ds[i].copy_(xs[i], non_blocking=True)
        for i in range(2):
            torch.cuda.current_stream().wait_stream(streams[i])
    else:  # 4 streams, 64 MB chunks
        for i in range(2):
            for h in range(2):
                s = streams[2 * i + h]
                s.wait_event(a)
                with torch.cuda.stream(s):
                    ds[i][h * n // 2:(h + 1) * n // 2].copy_(xs[i][h * n // 2:(h + 1) * n // 2],
                                                              non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return 2 * n / (a.elapsed_time(b) * 1e-3) / 1e9


for mode in ["1 stream", "2 streams", "4 streams"]:
    r = [run(mode) for _ in range(6)]
    print(f"H2D {mode}: {max(r):.1f} GB/s (best of 6), {sorted(r)[3]:.1f} median")
