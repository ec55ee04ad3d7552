"""pytest plugin (``-p tests._dropin_plugin``): run the REFERENCE's own tests with
``flexep.dispatch`` replaced by the drop-in ``paper_2407_04656_b200.dispatch`` -- the
one-import switch INTEGRATION.md describes.  The unmodified reference package comes from
``baseline/_ref`` (tools/install_reference.sh); its modules that imported the dispatcher
at import time (simulator, cli) are re-pointed as a maintainer's switch would."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

import flexep  # noqa: E402  (the reference, unmodified)
import flexep.cli  # noqa: E402
import flexep.simulator  # noqa: E402

from paper_2407_04656_b200 import dispatch as dropin  # noqa: E402

sys.modules["flexep.dispatch"] = dropin
flexep.dispatch = dropin
for mod in (flexep, flexep.simulator, flexep.cli):
    for name in ("ReplicaMatrix", "DispatchSchedule", "build_shuffle_index",
                 "compute_dispatch_schedule", "full_dispatch_matrices", "gather_load_matrix",
                 "simulate_all_to_all"):
        if hasattr(mod, name):
            setattr(mod, name, getattr(dropin, name))

CALLS = {"n": 0}
_orig = dropin._lib.call


def _count(name, *a):
    CALLS["n"] += 1
    return _orig(name, *a)


dropin._lib.call = _count


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"DROPIN liblz calls: {CALLS['n']}")
