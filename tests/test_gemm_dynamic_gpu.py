"""The grouped GEMM's dynamic tile scheduler (LZ_GEMM_DYNAMIC=1: atomic fetch + shared-
memory queue to every role of both CTAs, self-resetting per-launch counters) must give
the same results as the static schedule: the GEMM and layer parity tests run again in a
subprocess with it enabled (the policy is read once per process)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("policy", ["1", "2"])
def test_gemm_and_layer_parity_with_dynamic_scheduler(policy):
    env = dict(os.environ, LZ_GEMM_DYNAMIC=policy)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gemm_gpu.py"),
                        os.path.join(ROOT, "tests", "test_layer_gpu.py"),
                        os.path.join(ROOT, "tests", "test_loopback_gpu.py") +
                        "::test_loopback_fwd_bwd_matches_oracle"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
