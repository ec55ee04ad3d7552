"""Summarise ncu outputs brought back in gpurun_out/ into committed text files.

    python profiles/summarize.py <tag> [--launches gpurun_out/launches.csv]
                                 [--rep gpurun_out/gemm_full.ncu-rep ...]

Writes profiles/<tag>_launches.csv (per-kernel average of the launch list: cold,
serialised -- compare SHARES, not absolute times) and profiles/<tag>_kernels.csv
(selected `ncu --set full` metrics per captured launch).
"""

from __future__ import annotations

import collections
import csv
import io
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    # L2 side (the GEMMs' bound): bytes through the L2 slices, L2 -> SM
    # crossbar bytes, L2 throughput vs its peak, and the SM clock the kernel ran at
    "lts__t_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
]


def launches(path: str, tag: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:90]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    total = sum(tot.values())
    out = os.path.join(HERE, f"{tag}_launches.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "avg_us", "total_us", "share"])
        for n, t in sorted(tot.items(), key=lambda x: -x[1]):
            w.writerow([n, cnt[n], f"{t / cnt[n]:.1f}", f"{t:.1f}", f"{t / total:.3f}"])
    print("wrote", out)


def full(reps, tag: str) -> None:
    out = os.path.join(HERE, f"{tag}_kernels.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["report"] + METRICS)
        for rep in reps:
            txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                 text=True).stdout
            rows = list(csv.reader(io.StringIO(txt)))
            if len(rows) < 3:
                continue
            h, units = rows[0], rows[1]
            for r in rows[2:]:
                vals = []
                for m in METRICS:
                    if m in h:
                        i = h.index(m)
                        vals.append(f"{r[i]} {units[i]}".strip() if m != "Kernel Name"
                                    else r[i].split("(")[0])
                    else:
                        vals.append("")
                w.writerow([os.path.basename(rep)] + vals)
    print("wrote", out)


if __name__ == "__main__":
    tag = sys.argv[1]
    args = sys.argv[2:]
    reps = []
    i = 0
    while i < len(args):
        if args[i] == "--launches":
            launches(args[i + 1], tag)
            i += 2
        elif args[i] == "--rep":
            reps.append(args[i + 1])
            i += 2
        else:
            i += 1
    if reps:
        full(reps, tag)
