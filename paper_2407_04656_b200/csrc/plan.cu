// plan.cu -- K2: replica-split planning, bit-exact with the reference dispatcher.
//
// Restates (paths relative to /root/reference/pkg/src/flexep):
//   quota            dispatch.py:143-151   q_e = ceil(t_e / r_e), 0 if r_e == 0
//   _dispatch_row    dispatch.py:110-126   keep local up to q_e*R[e][i], split overflow
//   split_proportionally core.py:321-341   largest remainder, ties -> lower index
//   compute_dispatch_schedule dispatch.py:162-196 (send/recv sizes of one rank)
//   build_shuffle_index dispatch.py:199-237 / invert_permutation :240-244
//
// Launch sequence of lz_plan_dispatch (all on one stream, no host sync):
//   count_kernel  <<<B, 256>>>   per-block expert histogram of `routed` (smem atomics)
//   plan_kernel   <<<1, 1024>>>  quotas, D for all senders, send/recv sizes, receive
//                                layout, per-(e,j) slot tables, grid-wide exclusive
//                                scan of the block histograms (warp per expert)
//   slot_kernel   <<<B, 256>>>   stable per-expert rank m(p) (block base + warp
//                                __match_any_sync/popc), destination j(p), slot, dest row
#include "common.cuh"

namespace lz {

constexpr int kPlanThreads = 1024;
constexpr int kSlotThreads = 256;
constexpr int kSlotWarps = kSlotThreads / 32;
constexpr int kChunk = 1024;  // assignments per slot/count block
constexpr int kPerWarp = kChunk / kSlotWarps;  // 128 = 4 rounds of 32

typedef unsigned __int128 u128;

// One sender row of the dispatch matrix for one expert (dispatch.py:110-126).
// Returns false when the split would divide a positive overflow over all-zero
// residuals (core.py:333-335; unreachable for consistent inputs).
__device__ bool dispatch_row(int i, int N, const int32_t* __restrict__ t_row,
                             const int32_t* __restrict__ r_row, int64_t q, int32_t* out_row) {
  int64_t resid[LZ_MAX_RANKS];
  int64_t rem[LZ_MAX_RANKS];
  const int64_t cap_i = q * (int64_t)r_row[i];
  const int64_t t_i = t_row[i];
  const int64_t keep = t_i < cap_i ? t_i : cap_i;
  const int64_t over = t_i - keep;
  if (over == 0) {
    for (int j = 0; j < N; ++j) out_row[j] = (j == i) ? (int32_t)keep : 0;
    return true;
  }
  int64_t wsum = 0;
  for (int j = 0; j < N; ++j) {
    int64_t cap = q * (int64_t)r_row[j];
    int64_t t = t_row[j];
    resid[j] = (j == i) ? 0 : cap - (cap < t ? cap : t);
    wsum += resid[j];
  }
  if (wsum == 0) {
    for (int j = 0; j < N; ++j) out_row[j] = (j == i) ? (int32_t)keep : 0;
    return false;
  }
  int64_t given = 0;
  int64_t base[LZ_MAX_RANKS];
  for (int j = 0; j < N; ++j) {
    u128 prod = (u128)over * (u128)resid[j];
    u128 b = prod / (u128)wsum;
    base[j] = (int64_t)b;
    rem[j] = (int64_t)(prod - b * (u128)wsum);
    given += base[j];
  }
  const int64_t left = over - given;  // < number of non-zero remainders
  for (int j = 0; j < N; ++j) {
    int ahead = 0;
    for (int jj = 0; jj < N; ++jj)
      ahead += (rem[jj] > rem[j]) || (rem[jj] == rem[j] && jj < j);
    int64_t v = base[j] + (ahead < left ? 1 : 0) + (j == i ? keep : 0);
    out_row[j] = (int32_t)v;
  }
  return true;
}

__global__ void __launch_bounds__(kSlotThreads) count_kernel(const int32_t* __restrict__ routed,
                                                             int P, int E, int B,
                                                             int32_t* __restrict__ blk_counts,
                                                             int32_t* __restrict__ err) {
  extern __shared__ int32_t s_hist[];
  // wait BEFORE releasing the plan kernel: it then starts with T / R (written before this
  // kernel) complete and overlaps its table phases with this histogram
  pdl_wait();
  pdl_launch_dependents();
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
  __syncthreads();
  const int b = blockIdx.x;
  const int p0 = b * kChunk;
  bool bad = false;
  for (int q = threadIdx.x; q < kChunk; q += blockDim.x) {
    int p = p0 + q;
    if (p < P) {
      int e = __ldg(routed + p);
      if (e >= 0 && e < E)
        atomicAdd(&s_hist[e], 1);
      else
        bad = true;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(err, LZ_ERRF_EXPERT_ID);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) blk_counts[e * B + b] = s_hist[e];
}

// Exclusive scan over blocks of the per-block expert histograms (warp per expert),
// then the conservation check of build_shuffle_index (dispatch.py:213-229): the
// routed list must hold exactly expect[e * stride] assignments of expert e.
__device__ void scan_block_counts(const int32_t* blk_counts, int32_t* blk_base, int E, int B,
                                  const int32_t* expect, int stride, int32_t* err) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
  for (int e = warp; e < E; e += nwarps) {
    int32_t carry = 0;
    for (int b00 = 0; b00 < B; b00 += 32 * 8) {
      int32_t vv[8];   // up to 8 chunks of 32 block counts in flight before the scans
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b00 + u * 32 + lane;
        vv[u] = (b < B) ? blk_counts[e * B + b] : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b0 = b00 + u * 32;
        if (b0 >= B) break;
        const int b = b0 + lane;
        const int32_t v = vv[u];
        int32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int32_t w = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += w;
        }
        if (b < B) blk_base[e * B + b] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == 0 && carry != expect[e * stride]) atomicOr(err, LZ_ERRF_COUNTS);
  }
}

struct PlanArgs {
  const int32_t* T;
  const int32_t* R;
  int E, N, rank, align, P, B;
  int64_t* quota;
  int32_t* D;
  int32_t* send_sizes;
  int32_t* recv_sizes;
  int32_t* recv_counts;
  int32_t* recv_m;
  int32_t* recv_off;
  int32_t* recv_src_off;
  int32_t* recv_stage_off;    // [E][N] row of (source i, expert e) in the a2a staging buffer
  int32_t* recv_cnt;          // [E][N] D[i][e][rank]
  int32_t* err;
  const int32_t* blk_counts;  // [E][B]
  int32_t* blk_base;          // [E][B]
  int32_t* tab_pref;          // [E][N+1]  prefix of D[rank][e][:]
  int32_t* tab_sdelta;        // [E][N]    slot = m + sdelta
  int32_t* tab_ddelta;        // [E][N]    dest row = m + ddelta
  int d_smem;                 // T, R and D staged in shared memory (they fit)
  int cap_rows;               // > 0: rows of every rank's receive / return buffer
  int32_t* need_rows;         // optional: rows the largest receive / send side needs
};

// Single block.  Dynamic smem: int64 q[E] | int32 M[N][E] | int32 padoff[N][E+1]
// (+ int32 T[E][N] | R[E][N] | D[N][E][N] when d_smem: every later phase reads D from
// shared memory instead of re-reading its own global writes)
__global__ void __launch_bounds__(kPlanThreads) plan_kernel(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  // launched behind count_kernel (which waited for its own predecessor before releasing
  // this grid): T and R are complete; only the final scan needs count_kernel's block
  // histograms, so the wait for it is deferred to there
  pdl_launch_dependents();
  if (a.P == 0) pdl_wait();   // no count_kernel in front: wait for whatever wrote T / R
  const int E = a.E, N = a.N, rank = a.rank;
  int64_t* s_q = reinterpret_cast<int64_t*>(s_raw);
  int32_t* s_M = reinterpret_cast<int32_t*>(s_q + E);  // M[j][e] = sum_i D[i][e][j]
  int32_t* s_pad = s_M + N * E;                         // padoff[j][e], e in [0, E]
  int32_t* s_T = s_pad + N * (E + 1);
  int32_t* s_R = s_T + E * N;
  int32_t* s_D = s_R + E * N;
  const int tid = threadIdx.x;
  const int32_t* Tm = a.T;
  const int32_t* Rm = a.R;
  if (a.d_smem) {
    for (int x = tid; x < E * N; x += blockDim.x) {
      s_T[x] = a.T[x];
      s_R[x] = a.R[x];
    }
    __syncthreads();
    Tm = s_T;
    Rm = s_R;
  }

  // -- quotas (dispatch.py:143-151) -----------------------------------------
  for (int e = tid; e < E; e += blockDim.x) {
    int64_t t_e = 0, r_e = 0;
    for (int j = 0; j < N; ++j) {
      t_e += Tm[e * N + j];
      r_e += Rm[e * N + j];
    }
    int64_t q = 0;
    if (r_e > 0) q = (t_e + r_e - 1) / r_e;  // == ceil(float(t)/float(r)) for t < 2^52
    else if (t_e > 0) atomicOr(a.err, LZ_ERRF_UNROUTABLE);
    s_q[e] = q;
    if (a.quota) a.quota[e] = q;
  }
  __syncthreads();

  // -- all senders' rows (dispatch.py:152-159) --------------------------------
  for (int row = tid; row < N * E; row += blockDim.x) {
    const int i = row / E, e = row % E;
    dispatch_row(i, N, Tm + e * N, Rm + e * N, s_q[e],
                 (a.d_smem ? s_D : a.D) + (size_t)row * N);
  }
  __syncthreads();
  if (a.d_smem)
    for (int x = tid; x < N * E * N; x += blockDim.x) a.D[x] = s_D[x];

  const int32_t* D = a.d_smem ? s_D : a.D;
  auto Dat = [&](int i, int e, int j) { return D[((size_t)i * E + e) * N + j]; };

  // -- per-destination received counts and padded expert-major offsets -----------
  for (int x = tid; x < N * E; x += blockDim.x) {
    const int j = x / E, e = x % E;
    int32_t m = 0;
    for (int i = 0; i < N; ++i) m += Dat(i, e, j);
    s_M[j * E + e] = m;
  }
  __syncthreads();
  for (int j = tid; j < N; j += blockDim.x) {
    int32_t acc = 0;
    for (int e = 0; e < E; ++e) {
      s_pad[j * (E + 1) + e] = acc;
      int32_t m = s_M[j * E + e];
      acc += (m + a.align - 1) / a.align * a.align;
    }
    s_pad[j * (E + 1) + E] = acc;
    // send/recv sizes of `rank` (dispatch.py:178-184)
    int32_t s = 0, r = 0;
    for (int e = 0; e < E; ++e) {
      s += Dat(rank, e, j);
      r += Dat(j, e, rank);
    }
    a.send_sizes[j] = s;
    a.recv_counts[j] = r;
    a.recv_sizes[j] = (j == rank) ? 0 : r;
  }
  __syncthreads();

  // -- capacity of the exchange buffers: every rank evaluates the same plan, so every rank
  // takes the same decision.  Rank j receives padoff[j][E] rows; sender i's rows return to
  // its send slots (< sum_e T[e][i]).  On overflow nothing may be exchanged: the receive
  // layout becomes empty (no GEMM tile, no pad row) and slot_kernel keeps every row local.
  __shared__ int s_over;
  if (tid == 0) {
    int32_t need = 0;
    for (int j = 0; j < N; ++j) {
      need = max(need, s_pad[j * (E + 1) + E]);
      int32_t sent = 0;
      for (int e = 0; e < E; ++e) sent += Tm[e * N + j];
      need = max(need, sent);
    }
    const int over = a.cap_rows > 0 && need > a.cap_rows;
    if (over) atomicOr(a.err, LZ_ERRF_CAPACITY);
    if (a.need_rows) *a.need_rows = need;
    s_over = over;
  }
  __syncthreads();
  if (s_over)
    for (int x = tid; x < N * (E + 1); x += blockDim.x) s_pad[x] = 0;
  __syncthreads();

  // -- slot / destination tables for this rank's assignments --------------------
  for (int x = tid; x < E * N; x += blockDim.x) {
    const int e = x / N, j = x % N;
    int32_t pref = 0;
    for (int jj = 0; jj < j; ++jj) pref += Dat(rank, e, jj);
    int32_t sbase = 0;  // sum_{j'<j} s_j' + sum_{e'<e} D[rank][e'][j]
    for (int jj = 0; jj < j; ++jj)
      for (int ee = 0; ee < E; ++ee) sbase += Dat(rank, ee, jj);
    for (int ee = 0; ee < e; ++ee) sbase += Dat(rank, ee, j);
    int32_t dbase = s_pad[j * (E + 1) + e];  // rows of earlier senders on rank j
    for (int i = 0; i < rank; ++i) dbase += Dat(i, e, j);
    a.tab_sdelta[e * N + j] = sbase - pref;
    a.tab_ddelta[e * N + j] = dbase - pref;
    a.tab_pref[e * (N + 1) + j] = pref;
    if (j == N - 1) a.tab_pref[e * (N + 1) + N] = pref + Dat(rank, e, j);
  }
  // receive layout of `rank`
  for (int x = tid; x < E * N; x += blockDim.x) {
    const int e = x / N, i = x % N;
    int32_t off = s_pad[rank * (E + 1) + e];
    for (int ii = 0; ii < i; ++ii) off += Dat(ii, e, rank);
    a.recv_src_off[e * N + i] = s_over ? 0 : off;
    if (a.recv_stage_off) {
      int32_t st = 0;  // source-major blocks, expert-major inside a block
      for (int ii = 0; ii < i; ++ii)
        for (int ee = 0; ee < E; ++ee) st += Dat(ii, ee, rank);
      for (int ee = 0; ee < e; ++ee) st += Dat(i, ee, rank);
      a.recv_stage_off[e * N + i] = s_over ? 0 : st;
      a.recv_cnt[e * N + i] = s_over ? 0 : Dat(i, e, rank);
    }
  }
  for (int e = tid; e <= E; e += blockDim.x) {
    a.recv_off[e] = s_pad[rank * (E + 1) + e];
    if (e < E) a.recv_m[e] = s_over ? 0 : s_M[rank * E + e];
  }

  // -- grid-wide exclusive scan of block histograms, one warp per expert --------
  pdl_wait();
  if (a.P > 0) scan_block_counts(a.blk_counts, a.blk_base, E, a.B, a.T + rank, N, a.err);
}

__global__ void __launch_bounds__(kSlotThreads) slot_kernel(
    const int32_t* __restrict__ routed, int P, int E, int N, int B,
    const int32_t* __restrict__ blk_base, const int32_t* __restrict__ tab_pref,
    const int32_t* __restrict__ tab_sdelta, const int32_t* __restrict__ tab_ddelta,
    int32_t* __restrict__ slot, int32_t* __restrict__ gather, int32_t* __restrict__ dest_row,
    int32_t* __restrict__ dest_rank, int32_t* __restrict__ err, int rank, int cap_rows) {
  extern __shared__ int32_t s_cnt[];  // [kSlotWarps][E]
  pdl_prologue();
  const int b = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (cap_rows > 0 && (*(volatile int32_t*)err & LZ_ERRF_CAPACITY)) {
    // the exchange buffers are too small for this plan (plan_kernel): keep every row on
    // this rank at an in-bounds row, so the step's kernels run harmlessly and the host
    // grows the buffers and re-runs the step
    for (int q = threadIdx.x; q < kChunk; q += blockDim.x) {
      const int p = b * kChunk + q;
      if (p < P) {
        slot[p] = p % cap_rows;
        if (dest_row) dest_row[p] = p % cap_rows;
        if (dest_rank) dest_rank[p] = rank;
      }
    }
    return;
  }
  for (int x = threadIdx.x; x < kSlotWarps * E; x += blockDim.x) s_cnt[x] = 0;
  __syncthreads();
  const int p_warp = b * kChunk + warp * kPerWarp;
  int e_reg[kPerWarp / 32];
#pragma unroll
  for (int r = 0; r < kPerWarp / 32; ++r) {
    int p = p_warp + r * 32 + lane;
    int e = (p < P) ? __ldg(routed + p) : -1;
    if (e >= E) e = -1;
    e_reg[r] = e;
    if (e >= 0) atomicAdd(&s_cnt[warp * E + e], 1);
  }
  __syncthreads();
  // exclusive scan across warps per expert, seeded with the block's global base
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t acc = blk_base[e * B + b];
    for (int w = 0; w < kSlotWarps; ++w) {
      int32_t c = s_cnt[w * E + e];
      s_cnt[w * E + e] = acc;
      acc += c;
    }
  }
  __syncthreads();
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kPerWarp / 32; ++r) {
    const int p = p_warp + r * 32 + lane;
    const int e = e_reg[r];
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0) {
      const int32_t m = s_cnt[warp * E + e] + __popc(peers & lt);  // stable rank in expert e
      const int32_t* pref = tab_pref + e * (N + 1);
      // The routed list must hold exactly pref[N] assignments of expert e (checked in
      // scan_block_counts, dispatch.py:213-229); this kernel runs before the host can see
      // that flag, so an assignment beyond its expert's schedule row is flagged here and
      // written nowhere instead of walking past the row.
      if (m < pref[N]) {
        int j = 0;
        while (j + 1 < N && pref[j + 1] <= m) ++j;  // first D[e][0] -> rank 0, next D[e][1] -> 1, ...
        const int32_t s = m + tab_sdelta[e * N + j];
        if (s >= 0 && s < P) {
          slot[p] = s;
          gather[s] = p;
          if (dest_row) dest_row[p] = m + tab_ddelta[e * N + j];
          if (dest_rank) dest_rank[p] = j;
        } else {
          atomicOr(err, LZ_ERRF_COUNTS);
        }
      } else {
        atomicOr(err, LZ_ERRF_COUNTS);
      }
    }
    __syncwarp();
    if (e >= 0 && (peers & lt) == 0) s_cnt[warp * E + e] += __popc(peers);
    __syncwarp();
  }
}

}  // namespace lz

using namespace lz;

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

extern "C" lz_status lz_plan_workspace_bytes(int E, int N, int P, size_t* bytes) {
  if (!bytes || E < 1 || N < 1 || P < 0) return LZ_ERR_ARG;
  const size_t B = (size_t)(P + kChunk - 1) / kChunk;
  size_t n = 0;
  n += align_up(sizeof(int32_t) * E * B, 256) * 2;       // counts + base
  n += align_up(sizeof(int32_t) * E * (N + 1), 256);     // pref
  n += align_up(sizeof(int32_t) * E * N, 256) * 2;       // sdelta + ddelta
  *bytes = n + 256;
  return LZ_OK;
}

static lz_status check_EN(int E, int N) {
  if (E < 1 || N < 1) return LZ_ERR_ARG;
  if (N > LZ_MAX_RANKS || E > LZ_MAX_EXPERTS || E * N > LZ_MAX_EN) return LZ_ERR_UNSUPPORTED;
  return LZ_OK;
}

static size_t plan_smem(int E, int N, bool d_smem = false) {
  return sizeof(int64_t) * E + sizeof(int32_t) * (size_t)N * E + sizeof(int32_t) * (size_t)N * (E + 1) +
         (d_smem ? sizeof(int32_t) * ((size_t)2 * E * N + (size_t)N * E * N) : 0);
}
static bool plan_d_smem(int E, int N) { return plan_smem(E, N, true) <= 48 * 1024; }

extern "C" lz_status lz_plan_dispatch(const int32_t* T, const int32_t* R, int E, int N, int rank,
                                      const int32_t* routed, int P, int align, int cap_rows,
                                      int32_t* need_rows, int64_t* quota,
                                      int32_t* D, int32_t* send_sizes, int32_t* recv_sizes,
                                      int32_t* recv_counts, int32_t* slot, int32_t* gather,
                                      int32_t* dest_row, int32_t* dest_rank, int32_t* recv_m,
                                      int32_t* recv_off,
                                      int32_t* recv_src_off, int32_t* recv_stage_off,
                                      int32_t* recv_cnt, int32_t* err, void* ws,
                                      size_t ws_bytes, void* stream) {
  lz_status st = check_EN(E, N);
  if (st != LZ_OK) return st;
  if (rank < 0 || rank >= N || P < 0 || align < 1 || cap_rows < 0 || !T || !R || !D || !err || !send_sizes ||
      !recv_sizes || !recv_counts || !recv_m || !recv_off || !recv_src_off)
    return LZ_ERR_ARG;
  if (P > 0 && (!routed || !slot || !gather)) return LZ_ERR_ARG;
  if ((recv_stage_off == nullptr) != (recv_cnt == nullptr)) return LZ_ERR_ARG;
  size_t need = 0;
  lz_plan_workspace_bytes(E, N, P, &need);
  if (!ws || ws_bytes < need) return LZ_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const int B = (P + kChunk - 1) / kChunk;
  unsigned char* w = (unsigned char*)ws;
  w = (unsigned char*)align_up((size_t)w, 256);
  int32_t* blk_counts = (int32_t*)w;  w += align_up(sizeof(int32_t) * E * B, 256);
  int32_t* blk_base = (int32_t*)w;    w += align_up(sizeof(int32_t) * E * B, 256);
  int32_t* pref = (int32_t*)w;        w += align_up(sizeof(int32_t) * E * (N + 1), 256);
  int32_t* sdelta = (int32_t*)w;      w += align_up(sizeof(int32_t) * E * N, 256);
  int32_t* ddelta = (int32_t*)w;

  if (P > 0 && (st = lzh::launch(count_kernel, dim3(B), dim3(kSlotThreads), sizeof(int32_t) * E,
                                 s, 1, routed, P, E, B, blk_counts, err)) != LZ_OK)
    return st;
  PlanArgs a{T, R, E, N, rank, align, P, B, quota, D, send_sizes, recv_sizes, recv_counts,
             recv_m, recv_off, recv_src_off, recv_stage_off, recv_cnt, err, blk_counts,
             blk_base, pref, sdelta, ddelta, plan_d_smem(E, N) ? 1 : 0, cap_rows, need_rows};
  const size_t smem = plan_smem(E, N, a.d_smem != 0);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if ((st = lzh::launch(plan_kernel, dim3(1), dim3(kPlanThreads), smem, s, 1, a)) != LZ_OK)
    return st;
  if (P > 0)
    return lzh::launch(slot_kernel, dim3(B), dim3(kSlotThreads),
                       sizeof(int32_t) * kSlotWarps * E, s, 1, routed, P, E, N, B,
                       (const int32_t*)blk_base, (const int32_t*)pref, (const int32_t*)sdelta,
                       (const int32_t*)ddelta, slot, gather, dest_row, dest_rank, err, rank,
                       cap_rows);
  return LZ_OK;
}

// full_dispatch_matrices only: runs plan_kernel with rank 0 and scratch outputs
// living in a small internal device buffer is avoided -- callers wanting the
// sizes use lz_plan_dispatch.  Here only quota and D are produced.
__global__ void __launch_bounds__(kPlanThreads) matrices_kernel(const int32_t* T, const int32_t* R,
                                                                int E, int N, int64_t* quota,
                                                                int32_t* D, int32_t* err) {
  extern __shared__ int64_t s_q2[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t t_e = 0, r_e = 0;
    for (int j = 0; j < N; ++j) {
      t_e += T[e * N + j];
      r_e += R[e * N + j];
    }
    int64_t q = 0;
    if (r_e > 0) q = (t_e + r_e - 1) / r_e;
    else if (t_e > 0) atomicOr(err, LZ_ERRF_UNROUTABLE);
    s_q2[e] = q;
    if (quota) quota[e] = q;
  }
  __syncthreads();
  for (int row = threadIdx.x; row < N * E; row += blockDim.x) {
    const int i = row / E, e = row % E;
    dispatch_row(i, N, T + e * N, R + e * N, s_q2[e], D + (size_t)row * N);
  }
}

extern "C" lz_status lz_plan_matrices(const int32_t* T, const int32_t* R, int E, int N,
                                      int64_t* quota, int32_t* D, int32_t* err, void* stream) {
  lz_status st = check_EN(E, N);
  if (st != LZ_OK) return st;
  if (!T || !R || !D || !err) return LZ_ERR_ARG;
  matrices_kernel<<<1, kPlanThreads, sizeof(int64_t) * E, (cudaStream_t)stream>>>(T, R, E, N,
                                                                                 quota, D, err);
  return lzh::check_launch();
}

// build_shuffle_index from a schedule alone (send_counts = D[rank], E x N).
__global__ void __launch_bounds__(kPlanThreads) tables_kernel(const int32_t* send_counts, int E,
                                                              int N, int B,
                                                              const int32_t* blk_counts,
                                                              int32_t* blk_base, int32_t* pref,
                                                              int32_t* sdelta, int32_t* err) {
  extern __shared__ int32_t s_tot[];  // expected per-expert totals
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t t = 0;
    for (int j = 0; j < N; ++j) t += send_counts[e * N + j];
    s_tot[e] = t;
  }
  for (int x = threadIdx.x; x < E * N; x += blockDim.x) {
    const int e = x / N, j = x % N;
    int32_t p = 0;
    for (int jj = 0; jj < j; ++jj) p += send_counts[e * N + jj];
    int32_t sb = 0;
    for (int jj = 0; jj < j; ++jj)
      for (int ee = 0; ee < E; ++ee) sb += send_counts[ee * N + jj];
    for (int ee = 0; ee < e; ++ee) sb += send_counts[ee * N + j];
    sdelta[e * N + j] = sb - p;
    pref[e * (N + 1) + j] = p;
    if (j == N - 1) pref[e * (N + 1) + N] = p + send_counts[e * N + j];
  }
  __syncthreads();
  scan_block_counts(blk_counts, blk_base, E, B, s_tot, 1, err);
}

extern "C" lz_status lz_shuffle_index(const int32_t* send_counts, int E, int N,
                                      const int32_t* routed, int P, int32_t* slot,
                                      int32_t* gather, int32_t* err, void* ws, size_t ws_bytes,
                                      void* stream) {
  lz_status st = check_EN(E, N);
  if (st != LZ_OK) return st;
  if (P < 0 || !send_counts || !err) return LZ_ERR_ARG;
  if (P > 0 && (!routed || !slot || !gather)) return LZ_ERR_ARG;
  size_t need = 0;
  lz_plan_workspace_bytes(E, N, P, &need);
  if (!ws || ws_bytes < need) return LZ_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const int B = (P + kChunk - 1) / kChunk;
  unsigned char* w = (unsigned char*)align_up((size_t)ws, 256);
  int32_t* blk_counts = (int32_t*)w;  w += align_up(sizeof(int32_t) * E * B, 256);
  int32_t* blk_base = (int32_t*)w;    w += align_up(sizeof(int32_t) * E * B, 256);
  int32_t* pref = (int32_t*)w;        w += align_up(sizeof(int32_t) * E * (N + 1), 256);
  int32_t* sdelta = (int32_t*)w;
  if (P > 0) {
    count_kernel<<<B, kSlotThreads, sizeof(int32_t) * E, s>>>(routed, P, E, B, blk_counts, err);
    if ((st = lzh::check_launch()) != LZ_OK) return st;
  }
  tables_kernel<<<1, kPlanThreads, sizeof(int32_t) * E, s>>>(send_counts, E, N, B, blk_counts,
                                                             blk_base, pref, sdelta, err);
  if ((st = lzh::check_launch()) != LZ_OK) return st;
  if (P > 0) {
    slot_kernel<<<B, kSlotThreads, sizeof(int32_t) * kSlotWarps * E, s>>>(
        routed, P, E, N, B, blk_base, pref, sdelta, sdelta, slot, gather, nullptr, nullptr, err, 0,
        0);
    if ((st = lzh::check_launch()) != LZ_OK) return st;
  }
  return LZ_OK;
}

// Routing-history accumulator: one step's global per-expert load
// (row sums of the all-gathered T) into slot pos % W of a device ring, pos advanced on
// the device -- so the record is CUDA-graph safe.  The host reads the window only at a
// rebalance (simulator.py:342-351 window_loads; :642-644 trailing window of W steps).
__global__ void load_record_kernel(const int32_t* __restrict__ T, int E, int N,
                                   int64_t* __restrict__ ring, int W, int64_t* __restrict__ pos) {
  const int64_t p = *pos;
  const int64_t slot = p % W;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t s = 0;
    for (int j = 0; j < N; ++j) s += T[(size_t)e * N + j];
    ring[slot * E + e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) *pos = p + 1;
}

extern "C" lz_status lz_load_record(const int32_t* T, int E, int N, int64_t* ring, int W,
                                    int64_t* pos, void* stream) {
  lz_status st = check_EN(E, N);
  if (st != LZ_OK) return st;
  if (!T || !ring || !pos || W < 1) return LZ_ERR_ARG;
  load_record_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(T, E, N, ring, W, pos);
  return lzh::check_launch();
}
