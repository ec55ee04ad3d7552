"""ctypes binding of liblz.so (include/lz.h).  There is no fallback: if the
library is missing or fails to load, every entry point raises."""

from __future__ import annotations

import ctypes
import os
import threading

_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LZ_LIB_PATH") or os.path.join(_DIR, "liblz.so")  # override: A/B builds (tools/)

_vp, _i, _sz, _fp = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p

# name -> argtypes (restype int status unless listed in _RESTYPE)
_SIGS = {
    "lz_status_string": [_i],
    "lz_version": [],
    "lz_last_cuda_error": [],
    "lz_plan_matrices": [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp],
    "lz_plan_workspace_bytes": [_i, _i, _i, ctypes.POINTER(ctypes.c_size_t)],
    # T R E N rank routed P align | quota D send recv recv_counts slot gather dest_row
    # dest_rank recv_m recv_off recv_src_off recv_stage_off recv_cnt err ws | ws_bytes stream
    # ... align cap_rows need_rows | quota ...
    "lz_plan_dispatch": [_vp, _vp, _i, _i, _i, _vp, _i, _i, _i] + [_vp] * 17 + [_sz, _vp],
    "lz_set_control": [_vp],
    "lz_peer_barrier": [_vp, _i, _i, _vp, _vp, _vp],
    "lz_peer_barrier_colocated": [_vp, _i, _vp, _i, _vp, _vp, _vp],
    "lz_pack_p2p": [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp],
    "lz_combine_p2p": [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp],
    "lz_combine_bwd_p2p": [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp],
    "lz_dispatch_bwd_p2p": [_vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp,
                            _vp],
    "lz_shuffle_index": [_vp, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _sz, _vp],
    "lz_load_record": [_vp, _i, _i, _vp, _i, _vp, _vp],
    "lz_recovery_count": [_vp, _i, _i, _i, _vp, _vp],
    "lz_pack_p2p_ret": [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i, _vp,
                        _vp],
    "lz_combine_bwd_p2p_ret": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _i, _vp,
                               _vp, _vp],
    "lz_epoch_bump": [_vp, _vp],
    "lz_signal_peers": [_vp, _i, _i, _vp, _vp],
    "lz_grouped_gemm_arrival": [_vp, _vp, _vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp, _i,
                                _vp, _vp],
    "lz_grouped_gemm_scatter": [_vp, _vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i,
                                _i, _vp],
    "lz_gate_topk": [_vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp],
    "lz_router_gate": [_vp, _vp, _vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp],
    "lz_gate_bwd": [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp],
    "lz_invert_permutation": [_vp, _i, _vp, _vp],
    "lz_pack": [_vp, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp],
    "lz_copy_segments": [_vp, _vp, _i, _i, _vp, _vp, _vp, _i, _vp],
    "lz_combine": [_vp, _vp, _vp, _i, _i, _i, _vp, _vp],
    "lz_combine_bwd": [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp],
    "lz_dispatch_bwd": [_vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp],
    "lz_router_wgrad_ws_bytes": [_i, _i, _i],
    "lz_router_wgrad": [_vp, _vp, _i, _i, _i, _vp, _vp, _vp, _sz, _vp],
    "lz_gemm_set_cta_group": [_i],
    "lz_gemm_row_align": [],
    "lz_grouped_gemm": [_i, _vp, _vp, _vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _vp],
}
_RESTYPE = {"lz_status_string": ctypes.c_char_p, "lz_router_wgrad_ws_bytes": ctypes.c_size_t}

# header constants (include/lz.h)
LZ_OK, LZ_ERR_ARG, LZ_ERR_UNROUTABLE, LZ_ERR_CUDA, LZ_ERR_WORKSPACE, LZ_ERR_UNSUPPORTED = range(6)
LZ_ERRF_UNROUTABLE, LZ_ERRF_COUNTS, LZ_ERRF_EXPERT_ID, LZ_ERRF_CAPACITY = 1, 2, 4, 8
LZ_EPI_STORE, LZ_EPI_GELU, LZ_EPI_DGELU, LZ_EPI_SWIGLU, LZ_EPI_DSWIGLU = 0, 1, 2, 3, 4
LZ_K_MAJOR, LZ_MN_MAJOR = 0, 1
LZ_MAX_RANKS, LZ_MAX_EXPERTS, LZ_MAX_EN, LZ_MAX_TOPK = 64, 1024, 4096, 8


class LzError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn}: {msg} (status {status})")
        self.status = status


_lock = threading.Lock()
_handle = None


def load() -> ctypes.CDLL:
    """Load liblz.so once.  Raises if it is absent: the product has no CPU path."""
    global _handle
    if _handle is not None:
        return _handle
    with _lock:
        if _handle is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} not found: build it with `python -m paper_2407_04656_b200.build` "
                    "(the Lazarus B200 path has no CPU fallback)")
            h = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(h, name)
                fn.argtypes = args
                fn.restype = _RESTYPE.get(name, ctypes.c_int)
            _handle = h
    return _handle


def exported_symbols() -> list[str]:
    return list(_SIGS)


# kernels each entry point launches (for the bench's gpu_launches count)
_KERNELS = {"lz_plan_matrices": 1, "lz_plan_dispatch": 3, "lz_shuffle_index": 3,
            "lz_gate_topk": 1, "lz_router_gate": 1, "lz_gate_bwd": 1, "lz_invert_permutation": 1, "lz_pack": 1,
            "lz_copy_segments": 1, "lz_combine": 1, "lz_combine_bwd": 1, "lz_dispatch_bwd": 1,
            "lz_router_wgrad": 2, "lz_grouped_gemm": 1, "lz_pack_p2p": 1, "lz_combine_p2p": 1,
            "lz_combine_bwd_p2p": 1, "lz_dispatch_bwd_p2p": 1, "lz_load_record": 1,
            "lz_recovery_count": 1, "lz_pack_p2p_ret": 1, "lz_combine_bwd_p2p_ret": 1,
            "lz_grouped_gemm_scatter": 1, "lz_epoch_bump": 1, "lz_signal_peers": 1,
            "lz_grouped_gemm_arrival": 1, "lz_peer_barrier": 1,
            "lz_peer_barrier_colocated": 1}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    h = load()
    st = getattr(h, name)(*args)
    launch_count += _KERNELS.get(name, 0)
    if st != LZ_OK:
        msg = h.lz_status_string(st).decode()
        if st == LZ_ERR_CUDA:
            msg += f" (cudaError {h.lz_last_cuda_error()})"
        if st == LZ_ERR_ARG:
            raise ValueError(f"{name}: {msg}")
        raise LzError(name, st, msg)


def raw(name: str, *args):
    return getattr(load(), name)(*args)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ------------------------------------------------------------ watchdog control block

class Ctl(ctypes.Structure):
    """include/lz.h lz_ctl, in mapped pinned host memory (the host raises ``abort`` and
    reads the device-set causes without a device synchronisation)."""
    _fields_ = [("abort", ctypes.c_int32), ("timeout", ctypes.c_int32),
                ("aborted", ctypes.c_int32), ("watchdog", ctypes.c_int32),
                ("timeout_ns", ctypes.c_int64), ("reserved", ctypes.c_int64)]


_ctl_tensor = None
_ctl = None


def control(timeout_s: float | None = None) -> Ctl:
    """The process's control block (installed on first use; ``timeout_s`` sets the
    cross-rank wait budget, default 10 s).  Host-visible view over pinned memory the
    device reads and writes with system-scope accesses."""
    global _ctl_tensor, _ctl
    import torch
    if _ctl is None:
        t = torch.zeros(ctypes.sizeof(Ctl), dtype=torch.uint8).pin_memory()
        _ctl_tensor = t
        _ctl = Ctl.from_address(t.data_ptr())
        call("lz_set_control", ctypes.c_void_p(t.data_ptr()))
    if timeout_s is not None:
        _ctl.timeout_ns = int(timeout_s * 1e9)
    return _ctl


def control_status() -> dict:
    """Causes recorded by the device since the last :func:`control_reset` (no sync)."""
    c = control()
    return {"timeout": bool(c.timeout), "aborted": bool(c.aborted),
            "watchdog": bool(c.watchdog), "abort_raised": bool(c.abort)}


def control_abort() -> None:
    """Make every cross-rank wait in flight (and every later one) give up now."""
    control().abort = 1


def control_reset() -> None:
    c = control()
    c.abort = c.timeout = c.aborted = c.watchdog = 0
