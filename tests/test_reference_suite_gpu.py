"""The reference's OWN dispatcher tests, run against the drop-in.

``/root/reference/pkg/tests/test_dispatch.py`` (all 16 tests), the c07 fuzz
(``test_acceptance.py:243-292``, 10,000 instances) and c12 determinism
(``test_acceptance.py:581-617``: schedules, JSON forms and a whole simulator run whose
cost model now calls the device planner) execute unchanged with ``flexep.dispatch``
switched to ``paper_2407_04656_b200.dispatch`` (tests/_dropin_plugin.py).  They need the
reference copy in ``baseline/_ref`` (tools/install_reference.sh), which travels to the
GPU box; without it the test skips."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "reference_tests")


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="run tools/install_reference.sh first")
def test_reference_dispatch_tests_pass_on_the_dropin():
    targets = [os.path.join(SUITE, "test_dispatch.py"),
               os.path.join(SUITE, "test_acceptance.py") + "::test_c07_dispatch_conservation_and_balance",
               os.path.join(SUITE, "test_acceptance.py") + "::test_c12_determinism"]
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "-p", "tests._dropin_plugin", "--rootdir", SUITE, *targets],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "18 passed" in out, out[-2000:]
    calls = int(out.split("DROPIN liblz calls:")[1].split()[0])
    assert calls > 10_000, "the reference tests did not reach the device planner"
