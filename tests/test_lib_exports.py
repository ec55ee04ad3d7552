"""The C-ABI library loads and exports every symbol include/lz.h declares (CPU only)."""

import os
import re

from paper_2407_04656_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "lz.h")).read()
    return set(re.findall(r"^\s*(?:lz_status|const char\*|int|size_t)\s+(lz_\w+)\(", src, re.M))


def test_header_matches_binding():
    assert declared() == set(_lib.exported_symbols())


def test_library_loads_and_exports():
    h = _lib.load()
    for name in declared():
        assert hasattr(h, name), name
    assert h.lz_version() == 100
    assert h.lz_status_string(0) == b"ok"


def test_workspace_query_without_gpu():
    n = _lib.ctypes.c_size_t(0)
    _lib.call("lz_plan_workspace_bytes", 16, 8, 131072, _lib.ctypes.byref(n))
    assert n.value > 16 * 128 * 4
