"""One cfg2/cfg3 fwd+bwd step at N = 1 for ncu (bench.py's layer, plan and inputs).

    ncu --profile-from-start off ... python profiles/one_step.py [--config cfg2]

Three warm-up steps run outside the profiled range; the fourth is bracketed by
cudaProfilerStart/Stop, so ncu sees exactly one step's launches."""

from __future__ import annotations

import argparse
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402
from paper_2407_04656_b200 import ops  # noqa: E402
from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias  # noqa: E402
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    cfg = CONFIGS[ap.parse_args().config]
    E, k, d, dff, Tn = cfg["E"], cfg["k"], cfg["d"], cfg["dff"], cfg["tokens"]
    layer = MoELayer(d, dff, E, k, seed=0, router_bias=zipf_router_bias(E, cfg["s"], seed=0),
                     activation=cfg.get("act", "gelu"), router_std=1.28 / math.sqrt(d))
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    x = torch.randn(Tn, d, generator=g, device="cuda").bfloat16()
    dout = (torch.randn(Tn, d, generator=g, device="cuda") * 1e-2).bfloat16()
    hist = ops.router_gate(x, layer.wg.detach(), layer.bg.detach(), k)[3]
    layer.set_plan(replica_matrix(plan_for_loads(hist.long().cpu().tolist(), 1,
                                                 math.ceil(cfg["slot_factor"] * E), 2)))

    def step():
        layer.zero_grad(set_to_none=True)
        layer(x).backward(dout)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("one step done", flush=True)


if __name__ == "__main__":
    main()
