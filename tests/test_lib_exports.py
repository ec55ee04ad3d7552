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


def test_argument_errors_without_gpu():
    """Host-side argument checks return LZ_ERR_ARG / LZ_ERR_UNSUPPORTED before any device
    work (the Python layer maps them to ValueError / LzError), so they run on CPU."""
    h = _lib.load()
    A = _lib.LZ_ERR_ARG
    assert h.lz_plan_matrices(None, None, 0, 4, None, None, None, None) == A        # E = 0
    assert h.lz_router_gate(None, None, None, 16, 33, 8, 2, 0, None, None, None, None,
                            None) == A                                                # d % 32
    assert h.lz_router_gate(None, None, None, 16, 64, 8, 9, 0, None, None, None, None,
                            None) == A                                                # k > 8
    assert h.lz_grouped_gemm(0, None, None, None, None, 0, None, 0, 0, 256, 64, 0, 0, 0, 0, 0,
                             None) == A                                               # G = 0
    assert h.lz_recovery_count(None, 8, 64, 1, None, None) == A                       # N > 63
    assert h.lz_signal_peers(None, 0, 0, None, None) == A
    assert h.lz_load_record(None, 8, 2, None, 0, None, None) == A
    assert h.lz_pack_p2p_ret(None, 4, 64, 2, None, None, None, None, 0, None, None, None,
                             None, 0, None, None) == A                                # no peers
    try:
        _lib.call("lz_router_gate", None, None, None, 16, 33, 8, 2, 0, None, None, None, None,
                  None)
    except ValueError as e:
        assert "lz_router_gate" in str(e)
    else:
        raise AssertionError("LZ_ERR_ARG must raise ValueError")
