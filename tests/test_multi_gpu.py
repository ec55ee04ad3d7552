"""Multi-GPU parity under torchrun (skipped on a single-GPU box): tests/dist_layer_check.py
compares every rank's outputs, input grads and replica-group-summed expert grads with the
fp32 oracle on the gathered batch, for each exchange mode, then runs a periodic
rebalance and (N > 2) elastic shrinks."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{}, {"LZ_P2P_SCATTER": "0"}, {"LZ_EXCHANGE": "nccl"}])
def test_dist_layer(env):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(ROOT, "tests", "dist_layer_check.py"), "--rebalance", "--multilayer"]
    if n > 2 and not env:
        cmd.append("--elastic")
    if not env:
        cmd.append("--kill")
    r = subprocess.run(cmd, env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "DIST OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
