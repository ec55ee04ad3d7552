/*
 * lz.h -- C-ABI of liblz.so, the B200 (sm_100a) hot path of the Lazarus MoE layer
 * (arXiv 2407.04656): gating -> replica-split planning -> pack -> [all-to-all]
 * -> grouped expert FFN -> [all-to-all] -> combine, plus the backward kernels.
 *
 * The reference (flexep 0.1.0, pure Python) exposes the dispatcher as Python
 * functions; this header is the FFI a maintainer binds in their place (see
 * INTEGRATION.md for the ctypes stub).  Each entry point cites the reference
 * interface it replaces (paths relative to /root/reference/pkg/src/flexep).
 *
 * Conventions
 *   - every pointer is a DEVICE pointer unless stated; every call is asynchronous
 *     on `stream` (a cudaStream_t passed as void*), caller owns all memory,
 *     the library keeps no device state between calls (stateless, re-entrant);
 *   - T[e*N + j]  tokens routed to expert e originating on rank j  (E x N)
 *     R[e*N + j]  replicas of expert e on rank j, COMMUNICATOR-rank order (E x N)
 *     D[(i*E + e)*N + j] tokens of expert e sent by rank i to rank j (N x E x N)
 *   - routed assignments are flattened token-major: p = t*k + s;
 *   - bf16 tensors are row-major with the model dimension contiguous;
 *   - data-dependent errors (e.g. tokens routed to an expert without replicas)
 *     are reported through `err` (device int32 bit set, LZ_ERRF_*); the host reads
 *     it at its next synchronisation point and raises the reference's exception.
 */
#ifndef LZ_H_
#define LZ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LZ_OK = 0,
  LZ_ERR_ARG = 1,        /* host-side argument / shape error   (reference: ValueError)          */
  LZ_ERR_UNROUTABLE = 2, /* reserved for synchronous variants  (reference: UnroutableTokenError) */
  LZ_ERR_CUDA = 3,       /* CUDA launch / runtime error                                          */
  LZ_ERR_WORKSPACE = 4,  /* workspace too small                                                   */
  LZ_ERR_UNSUPPORTED = 5 /* shape outside the compiled limits                                     */
} lz_status;

/* device error-flag bits written into `err` */
#define LZ_ERRF_UNROUTABLE 1  /* t_e > 0 and r_e == 0          dispatch.py:147-150 */
#define LZ_ERRF_COUNTS 2      /* routed list disagrees with T  dispatch.py:213-229 */
#define LZ_ERRF_EXPERT_ID 4   /* routed expert id out of range dispatch.py:220-222 */
#define LZ_ERRF_CAPACITY 8    /* a rank's padded receive rows (or a sender's assignments)
                                 exceed the receive buffer: nothing was exchanged; the host
                                 grows the buffers and re-runs the step                  */

/* compiled limits */
#define LZ_MAX_RANKS 64
#define LZ_MAX_EXPERTS 1024
#define LZ_MAX_EN 4096 /* E*N */
#define LZ_MAX_TOPK 8

/* Watchdog / abort control block (process-wide; on a failure the enqueued
 * cross-rank waits time out and the step is discarded).  Every cross-rank wait of the
 * library (arrival flags of lz_grouped_gemm_arrival, lz_peer_barrier) gives up after
 * timeout_ns or as soon as the host raises `abort`, records why, and lets its kernel run
 * to completion on whatever data is present -- no kernel hangs and none traps; the host
 * discards the step.  Intra-kernel pipeline waits (a library bug, never a peer) record
 * `watchdog` after ~10 s and give up likewise.  Place the block in mapped pinned host
 * memory so the host can raise `abort` while kernels spin and poll the flags without a
 * device synchronisation.  Without a block (NULL) cross-rank waits are bounded by 10 s
 * and a stuck pipeline traps. */
typedef struct lz_ctl {
  int32_t abort;      /* host: non-zero -> every cross-rank wait gives up now            */
  int32_t timeout;    /* device: set to 1 when a cross-rank wait exceeded timeout_ns      */
  int32_t aborted;    /* device: set to 1 when a wait gave up because abort was raised    */
  int32_t watchdog;   /* device: set to 1 when an intra-kernel pipeline wait hit ~10 s    */
  int64_t timeout_ns; /* cross-rank wait budget (0: 10 s)                                 */
  int64_t reserved;
} lz_ctl;
/* Install (or with NULL remove) the control block; synchronous, call outside capture. */
lz_status lz_set_control(lz_ctl* ctl);

const char* lz_status_string(int status);
int lz_version(void);
int lz_last_cuda_error(void); /* cudaError_t of the last failed call on this thread */

/* ---------------------------------------------------------------- K2 planning */

/* Replaces full_dispatch_matrices (dispatch.py:129-159) + the quota computation
 * (dispatch.py:143-151): quota[E] (int64) and D for ALL senders, bit-exact with the
 * reference (largest-remainder split core.py:321-341, ties to the lower rank). */
lz_status lz_plan_matrices(const int32_t* T, const int32_t* R, int E, int N, int64_t* quota,
                           int32_t* D, int32_t* err, void* stream);

/* Workspace needed by lz_plan_dispatch for (E, N, P). */
lz_status lz_plan_workspace_bytes(int E, int N, int P, size_t* bytes);

/* Replaces compute_dispatch_schedule (dispatch.py:162-196) for `rank` plus
 * build_shuffle_index (dispatch.py:199-237) and invert_permutation (:240-244):
 *   quota[E], D[N*E*N]                   as lz_plan_matrices
 *   send_sizes[N]                        s_j incl. self                    (dispatch.py:178-180)
 *   recv_sizes[N]                        reference convention, self = 0    (dispatch.py:181-184)
 *   recv_counts[N]                       NCCL convention, self = D[r][*][r]
 *   slot[P]   send-buffer position of local assignment p (= invert_permutation(index))
 *   gather[P] local assignment at send slot s            (= build_shuffle_index result)
 *   dest_row[P] row of assignment p in its destination rank's expert-major receive
 *             buffer (segments padded to `align` rows, source-major inside an expert)
 *   dest_rank[P] (optional) the destination rank j of assignment p
 *   recv_m[E]        tokens of expert e this rank receives (incl. self)   (received[j][e][:] sum, :276-282)
 *   recv_off[E+1]    padded expert-major offsets of this rank's receive buffer
 *   recv_src_off[E*N] row where source i's tokens of expert e start on this rank
 *   recv_stage_off[E*N], recv_cnt[E*N] (optional, both or neither): where the
 *             (source i, expert e) segment sits in a plain all-to-all receive buffer
 *             (source-major, expert-major inside) and its length D[i][e][rank]
 * `routed` may be NULL (P = 0) to compute counts only.  Errors -> `err`.
 * cap_rows > 0: rows of every rank's exchange buffers.  When any rank's padded receive
 * rows or any sender's assignments exceed it, LZ_ERRF_CAPACITY is raised on EVERY rank
 * (all evaluate the same plan), the receive layout is empty and every assignment stays
 * local at row p % cap_rows -- the step runs harmlessly and the host grows the buffers to
 * *need_rows (optional output: the largest of those row counts) and re-runs it. */
lz_status lz_plan_dispatch(const int32_t* T, const int32_t* R, int E, int N, int rank,
                           const int32_t* routed, int P, int align, int cap_rows,
                           int32_t* need_rows, int64_t* quota, int32_t* D,
                           int32_t* send_sizes, int32_t* recv_sizes, int32_t* recv_counts,
                           int32_t* slot, int32_t* gather, int32_t* dest_row, int32_t* dest_rank,
                           int32_t* recv_m, int32_t* recv_off, int32_t* recv_src_off,
                           int32_t* recv_stage_off, int32_t* recv_cnt, int32_t* err, void* ws,
                           size_t ws_bytes, void* stream);

/* Replaces build_shuffle_index (dispatch.py:199-237) given only a schedule's
 * send_counts (E x N, = DispatchSchedule.send_counts): slot[P] and gather[P] as above;
 * validation errors (dispatch.py:213-229) -> `err`. ws as lz_plan_workspace_bytes. */
lz_status lz_shuffle_index(const int32_t* send_counts, int E, int N, const int32_t* routed, int P,
                           int32_t* slot, int32_t* gather, int32_t* err, void* ws,
                           size_t ws_bytes, void* stream);

/* Routing-history window: ring[(pos % W) * E + e] = sum_j T[e*N + j]; ++pos (device).
 * Replaces the reference's per-step load snapshot appended to the trailing window
 * (simulator.py:642-644); window_loads (simulator.py:342-351) = sum of the first
 * min(pos, W) ring rows // min(pos, W), computed by the host at a rebalance. */
lz_status lz_load_record(const int32_t* T, int E, int N, int64_t* ring, int W, int64_t* pos,
                         void* stream);

/* ------------------------------------------------------------------- K1 gating */

/* softmax over E logits, top-k (ties -> lower expert id), weights = top-k probs
 * (renorm = 0) or renormalised over the k (renorm = 1), per-rank expert
 * histogram hist[E] = T[:, rank] (the gather_load_matrix input, dispatch.py:95-107).
 * logits fp32 [Tn, E]. probs (fp32 [Tn, E]) may be NULL. */
lz_status lz_gate_topk(const float* logits, int Tn, int E, int k, int renorm, int32_t* idx,
                       float* w, float* probs, int32_t* hist, void* stream);

/* Fused router: logits = x[Tn, d] (bf16) . wg[E, d]^T (bf16) + bias[E] (fp32, may be
 * NULL), fp32 accumulate, then as lz_gate_topk.  d % 32 == 0, E <= 64; x and wg
 * 16-byte aligned (LZ_ERR_ARG otherwise).  A token's logits depend only on its row
 * (fixed accumulation order for a given d, E), never on Tn or its position. */
lz_status lz_router_gate(const void* x, const void* wg, const float* bias, int Tn, int d, int E,
                         int k, int renorm, int32_t* idx, float* w, float* probs, int32_t* hist,
                         void* stream);

/* Gate backward alone: dlogits[Tn, E] (fp32) from probs (fp32 [Tn, E]), idx and the
 * combine backward's dw [Tn, k] -- softmax + top-k (+ renorm) backward,
 * bit-identical to the dlogits lz_dispatch_bwd returns.  Lets the router weight gradient
 * start right after the combine backward.  probs / dlogits 16-byte aligned. */
lz_status lz_gate_bwd(const float* probs, const int32_t* idx, const float* dw, int Tn, int E,
                      int k, int renorm, float* dlogits, void* stream);

/* Replaces invert_permutation (dispatch.py:240-244): out[index[i]] = i. */
lz_status lz_invert_permutation(const int32_t* index, int n, int32_t* out, void* stream);

/* ----------------------------------------------------------- K3 pack / regroup */

/* out[row[t*k+s]] = x[t] (bf16 rows of d elements; d % 8 == 0).  When E > 0 the
 * padding rows of the expert-major layout (recv_m, recv_off) are zero-filled. */
lz_status lz_pack(const void* x, int Tn, int d, int k, const int32_t* row, void* out, int E,
                  const int32_t* recv_m, const int32_t* recv_off, void* stream);

/* Row-segment copy: for every segment g, rows [src[g], src[g]+cnt[g]) of `in` go to
 * rows [dst[g], ...) of `out` (regroups an all-to-all receive buffer into the
 * expert-major GEMM layout and back).  nseg segments, all arrays device int32. */
lz_status lz_copy_segments(const void* in, void* out, int d, int nseg, const int32_t* src,
                           const int32_t* dst, const int32_t* cnt, int max_cnt, void* stream);

/* ------------------------------------------------------------------ K7 combine */

/* out[t] = sum_s w[t,s] * y[row[t*k+s]]  (fixed s order, fp32 accumulate, bf16 out). */
lz_status lz_combine(const void* y, const int32_t* row, const float* w, int Tn, int d, int k,
                     void* out, void* stream);

/* ------------------------------------- fused dispatch/combine over NVLink peers */
/* Variants of pack / combine / combine_bwd / dispatch_bwd that move rows straight to
 * or from the destination rank's symmetric receive buffer through NVLink P2P
 * (`peers*[N]`: device array of each rank's buffer base address, e.g. from torch
 * symmetric memory), replacing send-buffer + NCCL all-to-all-v + regroup.  The caller
 * orders them with a cross-rank barrier (writes complete before the peer reads). */
lz_status lz_pack_p2p(const void* x, int Tn, int d, int k, const int32_t* dest_rank,
                      const int32_t* dest_row, const unsigned long long* peers, void* own, int E,
                      const int32_t* recv_m, const int32_t* recv_off, void* stream);
/* As lz_pack_p2p, and records in the owner's return map (symmetric, int64 per receive
 * row: ret_peers[owner][dest_row] = my_rank << 32 | ret_row[t*k + s]; own pad rows = -1)
 * where each row must go back to -- consumed by lz_grouped_gemm_scatter.  With ret_row =
 * the plan's send slot every (owner, expert) segment returns to a contiguous row range. */
lz_status lz_pack_p2p_ret(const void* x, int Tn, int d, int k, const int32_t* dest_rank,
                          const int32_t* dest_row, const unsigned long long* peers, void* own,
                          int E, const int32_t* recv_m, const int32_t* recv_off,
                          const unsigned long long* ret_peers, long long* ret_own, int my_rank,
                          const int32_t* ret_row, void* stream);
lz_status lz_combine_p2p(const unsigned long long* peers_y, const int32_t* dest_rank,
                         const int32_t* dest_row, const float* w, int Tn, int d, int k, void* out,
                         void* stream);
lz_status lz_combine_bwd_p2p(const void* dout, const unsigned long long* peers_y,
                             const unsigned long long* peers_dy, const int32_t* dest_rank,
                             const int32_t* dest_row, const float* w, int Tn, int d, int k,
                             float* dw, void* own_dy, int E, const int32_t* recv_m,
                             const int32_t* recv_off, void* stream);
/* As lz_combine_bwd_p2p with y read locally: assignment p's expert output is row
 * y_row[p] of this rank's return buffer y_ret (written by the owners'
 * lz_grouped_gemm_scatter); dy rows still go to the owners' buffers. */
lz_status lz_combine_bwd_p2p_ret(const void* dout, const void* y_ret, const int32_t* y_row,
                                 const unsigned long long* peers_dy, const int32_t* dest_rank,
                                 const int32_t* dest_row, const float* w, int Tn, int d, int k,
                                 float* dw, void* own_dy, int E, const int32_t* recv_m,
                                 const int32_t* recv_off, void* stream);
lz_status lz_dispatch_bwd_p2p(const unsigned long long* peers_dxe, const int32_t* dest_rank,
                              const int32_t* dest_row, int Tn, int d, int k, const float* probs,
                              const int32_t* idx, const float* dw, const void* wg, int E,
                              int renorm, void* dx, float* dlogits, void* stream);

/* -------------------------------------------------------------- K8 backward */

/* dy[row[t,s]] = w[t,s] * dout[t];  dw[t,s] = <dout[t], y[row[t,s]]>  (fp32).
 * Padding rows of the expert-major layout are zero-filled when E > 0. */
lz_status lz_combine_bwd(const void* dout, const void* y, const int32_t* row, const float* w,
                         int Tn, int d, int k, void* dy, float* dw, int E, const int32_t* recv_m,
                         const int32_t* recv_off, void* stream);

/* Gate backward + dispatch backward, fused per token:
 *   dlogits[t,:] from probs, idx, dw (softmax/top-k(/renorm) backward)
 *   dx[t] = sum_s dxe[row[t,s]] + dlogits[t,:] . wg
 * wgT is the router weight TRANSPOSED, bf16 [d, E] (E even; may be NULL); d % 64 == 0. */
lz_status lz_dispatch_bwd(const void* dxe, const int32_t* row, int Tn, int d, int k,
                          const float* probs, const int32_t* idx, const float* dw,
                          const void* wgT, int E, int renorm, void* dx, float* dlogits,
                          void* stream);

/* Router weight gradient: dwg[E, d] (fp32) = dlogits^T . x ; dbias[E] = sum_t dlogits.
 * ws >= lz_router_wgrad_ws_bytes(). */
size_t lz_router_wgrad_ws_bytes(int Tn, int d, int E);
lz_status lz_router_wgrad(const float* dlogits, const void* x, int Tn, int d, int E, float* dwg,
                          float* dbias, void* ws, size_t ws_bytes, void* stream);

/* ----------------------------------------------------- K4-K6 grouped expert GEMM */

/* Epilogues */
#define LZ_EPI_STORE 0     /* C = acc (bf16)                                   */
#define LZ_EPI_GELU 1      /* C = gelu(acc), AUX = gelu'(acc) (bf16; the backward factor)   */
#define LZ_EPI_DGELU 2     /* C = acc * AUX   (AUX as written by LZ_EPI_GELU)             */
/* Every AUX buffer (GELU/DGELU [rows, N]; SWIGLU/DSWIGLU [S | Q]) has the byte size of a
 * row-major bf16 [rows, W] matrix but a private 32x32-blocked layout (element (r, c) at
 * ((r/32)*(W/32) + c/32)*1024 + ((c%32)/8)*256 + (r%32)*8 + c%8) that keeps the
 * epilogue's accesses coalesced without shared-memory staging; it is produced and
 * consumed only by the forward / backward epilogue pair. */
#define LZ_EPI_SWIGLU 3    /* B rows = W1|W3 interleaved in 128-row blocks; with g|u = acc:
                              C[rows, N/2] = silu(g) * u, AUX[rows, N] = [silu(g) | u silu'(g)] */
#define LZ_EPI_DSWIGLU 4   /* acc = dA[rows, N]; AUX = LZ_EPI_SWIGLU's [S | Q] [rows, 2N];
                              C[rows, 2N] = [dA * Q | dA * S] = [dgate | dup]              */
/* Operand majors */
#define LZ_K_MAJOR 0
#define LZ_MN_MAJOR 1

/* Grouped GEMM on tcgen05/TMEM (TMA-fed, persistent, warp-specialised).
 * Groups g = 0..G-1 are described by the device array off[G+1] (row offsets,
 * every segment a multiple of 128 rows):
 *   mode 0 ("rows"):   C[off[g]:off[g+1], :N] = A[off[g]:off[g+1], :K] . B_g
 *                      A K-major [rows, K]; B_g = B[g*N:(g+1)*N, :K] (b_major = K) or
 *                      B[g*K:(g+1)*K, :N] (b_major = MN)
 *   mode 1 ("wgrad"):  C_g[M, N] = A[off[g]:off[g+1], :M]^T . B[off[g]:off[g+1], :N]
 *                      (both MN-major, variable K = segment length); C_g starts at row
 *                      g*c_group_rows + c_row_offset of C viewed as [*, N] (c_group_rows = 0
 *                      means M: dense [G, M, N]); lets dW1/dW2 interleave in one flat
 *                      per-expert gradient buffer that is all-reduced without copies
 * M, N, K multiples of lz_gemm_row_align() / 256 / 64; mode-0 segments multiples of
 * lz_gemm_row_align(); mode-1 segments multiples of 64; G <= 128. */
lz_status lz_grouped_gemm(int mode, const void* A, const void* B, void* C, void* aux, int G,
                          const int32_t* off, int rows_total, int M, int N, int K, int b_major,
                          int epilogue, int num_sms, int c_group_rows, int c_row_offset,
                          void* stream);

/* GEMM variant: 2 = CTA-pair kernel (tcgen05 cta_group::2, 256-row tiles; default),
 * 1 = single-CTA kernel (128-row tiles).  Returns the active value. */
int lz_gemm_set_cta_group(int cta_group);
/* Scatter variant of the mode-0 store GEMM (the multi-GPU expert FFN's last GEMM of each
 * direction): output row r is written -- straight from the epilogue registers, over
 * NVLink for remote ranks -- to row (ret_map[r] & 0xffffffff) of the buffer at
 * ret_peers[ret_map[r] >> 32] (rows of N bf16); ret_map[r] < 0 marks a pad row.  C is
 * not written (pass any valid [rows_total, N] buffer).  The rows return to the ranks that
 * dispatched them, so the combine / dispatch-backward read their own memory.
 * ret_peers (device) and ret_peers_host (host copy) hold the n_peers return buffers of
 * ret_rows rows each; 32-row chunks returning to consecutive rows of one rank (n_peers <=
 * 8) go out as TMA bulk-tensor stores, the rest as per-row stores. */
lz_status lz_grouped_gemm_scatter(const void* A, const void* B, void* C, int G,
                                  const int32_t* off, int rows_total, int N, int K, int b_major,
                                  int num_sms, const long long* ret_map,
                                  const unsigned long long* ret_peers,
                                  const unsigned long long* ret_peers_host, int n_peers,
                                  int ret_rows, void* stream);
/* Row alignment mode-0 group segments must have for the active variant (128 or 256). */
int lz_gemm_row_align(void);

/* ---------------------------------------------------------- recovery probability */

/* Number of failed-node sets F (|F| = k_failed, nodes 0..n_nodes-1) that leave every
 * expert with a surviving holder: holders[e] = bit mask of the nodes holding expert e
 * (E <= 1024, n_nodes <= 63).  *good (device u64) is overwritten asynchronously.
 * recovery probability = good / C(n_nodes, k_failed).  Replaces the Python enumeration
 * of reliability.py:68-96 (recovery_probability_exact) without its 10^6-subset cap. */
lz_status lz_recovery_count(const unsigned long long* holders, int E, int n_nodes, int k_failed,
                            unsigned long long* good, void* stream);

/* ------------------------------------------------- arrival flags (multi-GPU exchange) */

/* ++*epoch on the stream (one per layer step; every rank bumps its own counter). */
lz_status lz_epoch_bump(int* epoch, void* stream);
/* After this rank's dispatch kernel on the stream: flag_peers[j][my_rank] = *epoch for every
 * rank j < n (system-scope release after a system fence).  flag_peers: device table of
 * the n ranks' flag arrays (symmetric int32 [n]). */
lz_status lz_signal_peers(const unsigned long long* flag_peers, int n, int my_rank,
                          const int* epoch, void* stream);
/* Device-side cross-rank barrier on the stream (replaces the symmetric-memory barrier
 * between the exchange's remote writes and the reads that depend on them): ++*counter,
 * then flag_peers[j][my_rank] = *counter for every j < n (system fence + release store),
 * then wait until own_flags[i] >= *counter for every i < n (acquire).  Bounded by the
 * control block (lz_set_control): on timeout / abort it records the cause and returns. */
lz_status lz_peer_barrier(const unsigned long long* flag_peers, int n, int my_rank, int* counter,
                          const int* own_flags, void* stream);
/* The same barrier for n_local ranks that share ONE GPU (single-GPU loopback of the
 * multi-rank path), as ONE launch with one warp per co-hosted rank -- ranks that wait on
 * each other must never be separate launches on one GPU (nothing makes them co-resident).
 * Warp w acts as rank ranks[w] with its counter at counter_ptrs[w] and its own flag row at
 * own_flag_ptrs[w] (device tables); flag_peers as above. */
lz_status lz_peer_barrier_colocated(const unsigned long long* flag_peers, int n, const int* ranks,
                                    int n_local, const unsigned long long* counter_ptrs,
                                    const unsigned long long* own_flag_ptrs, void* stream);
/* Arrival-ordered mode-0 grouped GEMM (the first expert GEMM of each direction on N > 1):
 * as lz_grouped_gemm(mode 0), but the tiles lying entirely inside self_rows[2g] ..
 * self_rows[2g+1] (the rows this rank dispatched to itself) run first, and the producer
 * acquires flags[0..n_flags) >= *epoch before the first tile with other ranks' rows. */
lz_status lz_grouped_gemm_arrival(const void* A, const void* B, void* C, void* aux, int G,
                                  const int32_t* off, int rows_total, int N, int K, int b_major,
                                  int epilogue, int num_sms, const int32_t* self_rows,
                                  const int* flags, int n_flags, const int* epoch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LZ_H_ */
