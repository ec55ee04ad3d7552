"""Thin torch-tensor wrappers over the liblz C-ABI kernels (include/lz.h).

Every function launches on the current CUDA stream, allocates its outputs with the
torch caching allocator and never synchronises.  No CPU path exists: a missing
library or a non-CUDA tensor raises.
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import ptr

ALIGN = 256  # upper bound of the GEMM M tile (receive-buffer expert segments are padded to it)


def row_align() -> int:
    """Padding of expert segments required by the active grouped-GEMM variant."""
    return int(_lib.raw("lz_gemm_row_align"))


def set_gemm_cta_group(cg: int) -> int:
    return int(_lib.raw("lz_gemm_set_cta_group", cg))


def _s():
    return _lib.stream_ptr()


def _cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("liblz kernels take CUDA tensors only")


def router_gate(x, wg, bias, k: int, renorm: bool = False, probs: bool = True):
    """logits = x . wg^T + bias (fp32 acc) -> softmax/top-k.  Returns idx [T,k] int32,
    w [T,k] fp32, probs [T,E] fp32 (or None), hist [E] int32."""
    _cuda(x, wg, bias)
    Tn, d = x.shape
    E = wg.shape[0]
    dev = x.device
    idx = torch.empty((Tn, k), dtype=torch.int32, device=dev)
    w = torch.empty((Tn, k), dtype=torch.float32, device=dev)
    pr = torch.empty((Tn, E), dtype=torch.float32, device=dev) if probs else None
    hist = torch.empty(E, dtype=torch.int32, device=dev)
    _lib.call("lz_router_gate", ptr(x), ptr(wg), ptr(bias), Tn, d, E, k, int(renorm), ptr(idx),
              ptr(w), ptr(pr), ptr(hist), _s())
    return idx, w, pr, hist


def gate_topk(logits, k: int, renorm: bool = False, probs: bool = True):
    _cuda(logits)
    Tn, E = logits.shape
    dev = logits.device
    idx = torch.empty((Tn, k), dtype=torch.int32, device=dev)
    w = torch.empty((Tn, k), dtype=torch.float32, device=dev)
    pr = torch.empty((Tn, E), dtype=torch.float32, device=dev) if probs else None
    hist = torch.empty(E, dtype=torch.int32, device=dev)
    _lib.call("lz_gate_topk", ptr(logits.float().contiguous()), Tn, E, k, int(renorm), ptr(idx),
              ptr(w), ptr(pr), ptr(hist), _s())
    return idx, w, pr, hist


def pack(x, row, k: int, out, recv_m=None, recv_off=None):
    """out[row[t*k+s]] = x[t]; zero-fills the padding rows when recv_m/recv_off given."""
    _cuda(x, row, out)
    Tn, d = x.shape
    E = 0 if recv_m is None else recv_m.numel()
    _lib.call("lz_pack", ptr(x), Tn, d, k, ptr(row), ptr(out), E, ptr(recv_m), ptr(recv_off),
              _s())
    return out


def zero_pad_rows(buf, recv_m, recv_off):
    d = buf.shape[1]
    _lib.call("lz_pack", None, 0, d, 1, None, ptr(buf), recv_m.numel(), ptr(recv_m),
              ptr(recv_off), _s())


def copy_segments(src_buf, dst_buf, src_off, dst_off, cnt, max_cnt: int):
    d = src_buf.shape[1]
    _lib.call("lz_copy_segments", ptr(src_buf), ptr(dst_buf), d, cnt.numel(), ptr(src_off),
              ptr(dst_off), ptr(cnt), int(max_cnt), _s())
    return dst_buf


def combine(y, row, w, k: int, out=None):
    _cuda(y, row, w)
    Tn = w.shape[0]
    d = y.shape[1]
    if out is None:
        out = torch.empty((Tn, d), dtype=torch.bfloat16, device=y.device)
    _lib.call("lz_combine", ptr(y), ptr(row), ptr(w), Tn, d, k, ptr(out), _s())
    return out


def combine_bwd(dout, y, row, w, k: int, dy, recv_m=None, recv_off=None):
    """dy[row[t,s]] = w[t,s] dout[t] (pads zeroed); returns dw [T,k] fp32."""
    _cuda(dout, y, row, w, dy)
    Tn, d = dout.shape
    dw = torch.empty((Tn, k), dtype=torch.float32, device=dout.device)
    E = 0 if recv_m is None else recv_m.numel()
    _lib.call("lz_combine_bwd", ptr(dout), ptr(y), ptr(row), ptr(w), Tn, d, k, ptr(dy), ptr(dw),
              E, ptr(recv_m), ptr(recv_off), _s())
    return dw


def dispatch_bwd(dxe, row, probs, idx, dw, wg, renorm: bool, Tn: int):
    _cuda(dxe, row, probs, idx, dw, wg)
    d = dxe.shape[1]
    k = idx.shape[1]
    E = probs.shape[1]
    dx = torch.empty((Tn, d), dtype=torch.bfloat16, device=dxe.device)
    dlog = torch.empty((Tn, E), dtype=torch.float32, device=dxe.device)
    wgT = None if wg is None else wg.t().contiguous()  # [d, E], experts contiguous
    _lib.call("lz_dispatch_bwd", ptr(dxe), ptr(row), Tn, d, k, ptr(probs), ptr(idx), ptr(dw),
              ptr(wgT), E, int(renorm), ptr(dx), ptr(dlog), _s())
    return dx, dlog


def gate_bwd(probs, idx, dw, renorm: bool):
    """dlogits [Tn, E] of the gate (softmax / top-k backward) -- bit-identical to the
    dlogits dispatch_bwd returns, available right after the combine backward."""
    _cuda(probs, idx, dw)
    Tn, E = probs.shape
    k = idx.shape[1]
    dlog = torch.empty((Tn, E), dtype=torch.float32, device=probs.device)
    _lib.call("lz_gate_bwd", ptr(probs), ptr(idx), ptr(dw), Tn, E, k, int(renorm), ptr(dlog),
              _s())
    return dlog


def router_wgrad(dlogits, x, with_bias: bool = True):
    _cuda(dlogits, x)
    Tn, d = x.shape
    E = dlogits.shape[1]
    dwg = torch.empty((E, d), dtype=torch.float32, device=x.device)
    db = torch.empty(E, dtype=torch.float32, device=x.device) if with_bias else None
    nbytes = int(_lib.raw("lz_router_wgrad_ws_bytes", Tn, d, E))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    _lib.call("lz_router_wgrad", ptr(dlogits), ptr(x), Tn, d, E, ptr(dwg), ptr(db), ptr(ws),
              nbytes, _s())
    return dwg, db


# Optional timing hook: when set to a list, every grouped-GEMM launch appends a
# (start, end) pair of CUDA events recorded on the launching stream (bench.py).  Under
# CUDA-graph capture set GEMM_EVENTS_EXTERNAL: the events become event-record nodes of
# the graph and time the GEMMs of every replay.
GEMM_EVENTS: list | None = None
GEMM_EVENTS_EXTERNAL = False


def _gemm(*args, fn: str = "lz_grouped_gemm"):
    if GEMM_EVENTS is None:
        _lib.call(fn, *args)
        return
    a = torch.cuda.Event(enable_timing=True, external=GEMM_EVENTS_EXTERNAL)
    b = torch.cuda.Event(enable_timing=True, external=GEMM_EVENTS_EXTERNAL)
    a.record()
    _lib.call(fn, *args)
    b.record()
    GEMM_EVENTS.append((a, b))


def grouped_gemm_rows(A, B, off, C, *, b_major=_lib.LZ_K_MAJOR, epilogue=_lib.LZ_EPI_STORE,
                      aux=None, num_sms: int = 0):
    """C[off[g]:off[g+1]] = A[off[g]:off[g+1]] . B_g (+ fused epilogue).
    A [rows, K]; B [G, N, K] (K-major) or [G, K, N] (MN-major); C [rows, N]."""
    _cuda(A, B, off, C, aux)
    rows, K = A.shape
    G = off.numel() - 1
    N = B.shape[1] if b_major == _lib.LZ_K_MAJOR else B.shape[2]
    _gemm(0, ptr(A), ptr(B), ptr(C), ptr(aux), G, ptr(off), rows, 0, N, K, b_major, epilogue,
          num_sms, 0, 0, _s())
    return C


def aux_rows(aux: torch.Tensor) -> torch.Tensor:
    """The epilogue aux streams (GELU: gelu'(h); SwiGLU: S | Q -- written by a forward
    epilogue, read only by the matching backward one) are stored in a private
    32x32-blocked layout that keeps the epilogue's global accesses coalesced without
    shared-memory staging (csrc/gemm.cu aux_block).  Row-major view of it (tests /
    debugging).  aux: [rows, W], rows % 32 == 0, W % 32 == 0."""
    R, N = aux.shape
    return aux.reshape(R // 32, N // 32, 4, 32, 8).permute(0, 3, 1, 2, 4).reshape(R, N)


def aux_blocked(rows_major: torch.Tensor) -> torch.Tensor:
    """Inverse of :func:`aux_rows`."""
    R, N = rows_major.shape
    return rows_major.reshape(R // 32, 32, N // 32, 4, 8).permute(0, 2, 3, 1, 4).reshape(R, N)


def grouped_gemm_scatter(A, B, off, C, ret_map, ret_peers, ret_peers_host, ret_rows: int, *,
                         b_major=_lib.LZ_K_MAJOR, num_sms: int = 0):
    """Mode-0 store GEMM whose output row r goes to row (ret_map[r] & 0xffffffff) of the
    return buffer of rank ret_map[r] >> 32 (TMA stores for contiguous 32-row chunks, per-row
    stores otherwise; NVLink for remote ranks); -1 = pad.  ret_peers: device int64 table of
    the buffers, ret_peers_host: the same addresses as Python ints, ret_rows: their rows.
    C ([rows, N], not written) only sizes the launch."""
    import ctypes
    _cuda(A, B, off, C, ret_map, ret_peers)
    rows, K = A.shape
    G = off.numel() - 1
    N = B.shape[1] if b_major == _lib.LZ_K_MAJOR else B.shape[2]
    host = (ctypes.c_ulonglong * max(1, len(ret_peers_host)))(*ret_peers_host)
    _gemm(ptr(A), ptr(B), ptr(C), G, ptr(off), rows, N, K, b_major, num_sms, ptr(ret_map),
          ptr(ret_peers), ctypes.cast(host, ctypes.c_void_p), len(ret_peers_host), int(ret_rows),
          _s(), fn="lz_grouped_gemm_scatter")
    return C


def grouped_gemm_arrival(A, B, off, C, self_rows, flags, epoch, *, b_major=_lib.LZ_K_MAJOR,
                         epilogue=_lib.LZ_EPI_STORE, aux=None, num_sms: int = 0):
    """grouped_gemm_rows whose tiles made of this rank's own rows (self_rows [G, 2]) run
    first; the rest wait for the senders' arrival flags (flags [N] >= *epoch)."""
    _cuda(A, B, off, C, self_rows, flags, epoch, aux)
    rows, K = A.shape
    G = off.numel() - 1
    N = B.shape[1] if b_major == _lib.LZ_K_MAJOR else B.shape[2]
    _gemm(ptr(A), ptr(B), ptr(C), ptr(aux), G, ptr(off), rows, N, K, b_major, epilogue, num_sms,
          ptr(self_rows), ptr(flags), flags.numel(), ptr(epoch), _s(),
          fn="lz_grouped_gemm_arrival")
    return C


def epoch_bump(epoch) -> None:
    _lib.call("lz_epoch_bump", ptr(epoch), _s())


def peer_barrier(flag_peers, n: int, my_rank: int, counter, own_flags, stream=None) -> None:
    """Device-side cross-rank barrier (bounded by the watchdog control block)."""
    _lib.call("lz_peer_barrier", ptr(flag_peers), int(n), int(my_rank), ptr(counter),
              ptr(own_flags), _lib.stream_ptr(stream))


def signal_peers(flag_peers, n: int, my_rank: int, epoch) -> None:
    """Publish this step's epoch in every rank's arrival-flag slot for this sender."""
    _lib.call("lz_signal_peers", ptr(flag_peers), int(n), int(my_rank), ptr(epoch), _s())


def grouped_gemm_wgrad(A, B, off, C, num_sms: int = 0, c_group_rows: int = 0,
                       c_row_offset: int = 0):
    """C_g = A[off[g]:off[g+1]]^T . B[off[g]:off[g+1]]; A [rows, M], B [rows, N].
    C is [G, M, N] (default) or any buffer where C_g starts at row g*c_group_rows +
    c_row_offset of C viewed as [*, N]."""
    _cuda(A, B, off, C)
    rows, M = A.shape
    N = B.shape[1]
    G = off.numel() - 1
    _gemm(1, ptr(A), ptr(B), ptr(C), None, G, ptr(off), rows, M, N, 0, _lib.LZ_MN_MAJOR,
          _lib.LZ_EPI_STORE, num_sms, c_group_rows, c_row_offset, _s())
    return C


# ------------------------------------------------- fused exchange over NVLink peers

def pack_p2p(x, dest_rank, dest_row, k: int, peers, own, recv_m, recv_off):
    """x rows -> their destination rank's symmetric receive buffer (P2P stores)."""
    Tn, d = x.shape
    _lib.call("lz_pack_p2p", ptr(x), Tn, d, k, ptr(dest_rank), ptr(dest_row), ptr(peers),
              ptr(own), recv_m.numel(), ptr(recv_m), ptr(recv_off), _s())


def combine_p2p(peers_y, dest_rank, dest_row, w, k: int, d: int, out=None):
    Tn = w.shape[0]
    if out is None:
        out = torch.empty((Tn, d), dtype=torch.bfloat16, device=w.device)
    _lib.call("lz_combine_p2p", ptr(peers_y), ptr(dest_rank), ptr(dest_row), ptr(w), Tn, d, k,
              ptr(out), _s())
    return out


def combine_bwd_p2p(dout, peers_y, peers_dy, dest_rank, dest_row, w, k: int, own_dy, recv_m,
                    recv_off):
    Tn, d = dout.shape
    dw = torch.empty((Tn, k), dtype=torch.float32, device=dout.device)
    _lib.call("lz_combine_bwd_p2p", ptr(dout), ptr(peers_y), ptr(peers_dy), ptr(dest_rank),
              ptr(dest_row), ptr(w), Tn, d, k, ptr(dw), ptr(own_dy), recv_m.numel(), ptr(recv_m),
              ptr(recv_off), _s())
    return dw


def dispatch_bwd_p2p(peers_dxe, dest_rank, dest_row, probs, idx, dw, wg, renorm: bool, Tn: int,
                     d: int):
    k = idx.shape[1]
    E = probs.shape[1]
    dx = torch.empty((Tn, d), dtype=torch.bfloat16, device=probs.device)
    dlog = torch.empty((Tn, E), dtype=torch.float32, device=probs.device)
    wgT = None if wg is None else wg.t().contiguous()
    _lib.call("lz_dispatch_bwd_p2p", ptr(peers_dxe), ptr(dest_rank), ptr(dest_row), Tn, d, k,
              ptr(probs), ptr(idx), ptr(dw), ptr(wgT), E, int(renorm), ptr(dx), ptr(dlog), _s())
    return dx, dlog


def pack_p2p_ret(x, dest_rank, dest_row, k: int, peers, own, recv_m, recv_off, ret_peers,
                 ret_own, my_rank: int, ret_row):
    """pack_p2p + the owners' return map (rank << 32 | ret_row[assignment]) for the scatter
    GEMM (ret_row = the plan's send slot)."""
    Tn, d = x.shape
    _lib.call("lz_pack_p2p_ret", ptr(x), Tn, d, k, ptr(dest_rank), ptr(dest_row), ptr(peers),
              ptr(own), recv_m.numel(), ptr(recv_m), ptr(recv_off), ptr(ret_peers),
              ptr(ret_own), int(my_rank), ptr(ret_row), _s())


def combine_bwd_p2p_ret(dout, y_ret, y_row, peers_dy, dest_rank, dest_row, w, k: int, own_dy,
                        recv_m, recv_off):
    """combine backward with y read from this rank's own return buffer at rows y_row."""
    Tn, d = dout.shape
    dw = torch.empty((Tn, k), dtype=torch.float32, device=dout.device)
    _lib.call("lz_combine_bwd_p2p_ret", ptr(dout), ptr(y_ret), ptr(y_row), ptr(peers_dy),
              ptr(dest_rank), ptr(dest_row), ptr(w), Tn, d, k, ptr(dw), ptr(own_dy),
              recv_m.numel(), ptr(recv_m), ptr(recv_off), _s())
    return dw


if "LZ_GEMM_CTA" in __import__("os").environ:  # A/B switch for the GEMM variant
    set_gemm_cta_group(int(__import__("os").environ["LZ_GEMM_CTA"]))
