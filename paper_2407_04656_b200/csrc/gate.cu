// gate.cu -- K1: gating softmax / top-k (+ fused router GEMM) and per-rank histogram.
//
// No reference code exists for this stage; semantics are
// restated from PAPER.md:94-95 ("a trainable gate network routes each token to
// only the top-k experts") with the reference's tie rule (lower id wins, as in
// allocation.py:94, placement.py:131, core.py:339).  Selection is done on the
// fp32 logits (exact), so the routed expert ids are bit-exact against the CPU
// oracle for identical logits; probabilities/weights carry fp32 rounding only.
//
// hist[e] is this rank's column T[:, rank] of the load matrix that the
// all-gather assembles (gather_load_matrix, dispatch.py:95-107).
#include "common.cuh"

namespace lz {

// Softmax + top-k for one token whose E logits are at `lg` (smem or global).
// KK > 0: compile-time k (the running top-k lives in registers); KK == 0: any k <= 8.
// Insertion keeps the list sorted by value; a new value is inserted only when strictly
// greater than an entry, so ties keep the lower expert id.
template <int KK>
__device__ __forceinline__ void finish_token_k(const float* lg, int E, int k, int renorm,
                                               int32_t* __restrict__ idx_out,
                                               float* __restrict__ w_out,
                                               float* __restrict__ probs_out,
                                               int32_t* s_hist) {
  constexpr int KM = KK > 0 ? KK : LZ_MAX_TOPK;
  const int kk = KK > 0 ? KK : k;
  int sel[KM];
  float sv[KM];
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    sel[s] = -1;
    sv[s] = -INFINITY;
  }
  float mx = -INFINITY;
  for (int e = 0; e < E; ++e) {
    const float v = lg[e];
    mx = fmaxf(mx, v);
    if (KK > 0) {
      // carry insertion over compile-time positions (registers only)
      bool ins = false;
      float cv = v;
      int ci = e;
#pragma unroll
      for (int p = 0; p < KM; ++p) {
        const bool here = !ins && (cv > sv[p] || sel[p] < 0);
        if (ins || here) {
          const float tv = sv[p];
          const int ti = sel[p];
          sv[p] = cv;
          sel[p] = ci;
          cv = tv;
          ci = ti;
          ins = true;
        }
      }
    } else if (v > sv[kk - 1] || sel[kk - 1] < 0) {
      int pos = kk - 1;
      while (pos > 0 && (v > sv[pos - 1] || sel[pos - 1] < 0)) {
        sv[pos] = sv[pos - 1];
        sel[pos] = sel[pos - 1];
        --pos;
      }
      sv[pos] = v;
      sel[pos] = e;
    }
  }
  float sum = 0.f;
  for (int e = 0; e < E; ++e) sum += expf(lg[e] - mx);
  const float inv = 1.f / sum;
  if (probs_out)
    for (int e = 0; e < E; ++e) probs_out[e] = expf(lg[e] - mx) * inv;
  float ps[KM];
  float psum = 0.f;
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    if (s < kk) {
      ps[s] = expf(sv[s] - mx) * inv;
      psum += ps[s];
    }
  }
  const float rn = renorm ? 1.f / psum : 1.f;
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    if (s < kk) {
      idx_out[s] = sel[s];
      w_out[s] = ps[s] * rn;
      atomicAdd(&s_hist[sel[s]], 1);
    }
  }
}

__device__ __forceinline__ void finish_token(const float* lg, int E, int k, int renorm,
                                             int32_t* __restrict__ idx_out,
                                             float* __restrict__ w_out,
                                             float* __restrict__ probs_out,
                                             int32_t* s_hist) {
  if (k == 2) finish_token_k<2>(lg, E, k, renorm, idx_out, w_out, probs_out, s_hist);
  else if (k == 1) finish_token_k<1>(lg, E, k, renorm, idx_out, w_out, probs_out, s_hist);
  else finish_token_k<0>(lg, E, k, renorm, idx_out, w_out, probs_out, s_hist);
}

// Logits staged through shared memory with coalesced loads (a block owns `tpb` whole
// logit rows, tpb * E <= 16K floats), then one thread per token runs the softmax/top-k on
// its (padded) smem row -- direct per-thread row reads were 32-way uncoalesced.
__global__ void __launch_bounds__(256) gate_topk_kernel(const float* __restrict__ logits, int Tn,
                                                        int E, int k, int renorm, int tpb,
                                                        int32_t* __restrict__ idx,
                                                        float* __restrict__ w,
                                                        float* __restrict__ probs,
                                                        int32_t* __restrict__ hist) {
  extern __shared__ float g_smem[];
  const int ld = E + 1;                                   // padded row (bank spread)
  float* s_lg = g_smem;                                   // [tpb][E + 1]
  int32_t* s_hist = reinterpret_cast<int32_t*>(g_smem + (size_t)tpb * ld);
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
  const long t0 = (long)blockIdx.x * tpb;
  const int nt = (int)min((long)tpb, (long)Tn - t0);
  const float* src = logits + t0 * E;
  {
    // warp per row, coalesced, asynchronous (cp.async: no register round trip, so the
    // loads of all rows are in flight together), no index division
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(s_lg);
    for (int r = threadIdx.x >> 5; r < nt; r += nw)
      for (int e = lane; e < E; e += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s0 + (uint32_t)(r * ld + e) * 4u),
                     "l"(src + (size_t)r * E + e)
                     : "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  if (E >= 16 && k <= 2) {
    // 8 lanes per token, each over every 8th expert: local max / sum / top-2, then
    // butterfly merges (ties -> lower id, as the sequential insertion)
    constexpr int L = 8;
    const int lane = threadIdx.x & 31, sub = lane & (L - 1);
    const unsigned gmask = 0xffffffffu;
    for (int ti0 = threadIdx.x / L; ti0 < ((nt + 3) & ~3); ti0 += blockDim.x / L) {
      // every lane of the warp iterates together (shuffles need the full warp)
      const bool live = ti0 < nt;
      const float* lg = s_lg + (size_t)(live ? ti0 : 0) * ld;
      float v1 = -INFINITY, v2 = -INFINITY, mx = -INFINITY;
      int i1 = 0x7fffffff, i2 = 0x7fffffff;
      for (int e = sub; e < E; e += L) {
        const float v = lg[e];
        mx = fmaxf(mx, v);
        if (v > v1) { v2 = v1; i2 = i1; v1 = v; i1 = e; }
        else if (v > v2) { v2 = v; i2 = e; }
      }
#pragma unroll
      for (int o = 1; o < L; o <<= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, o));
        const float w1 = __shfl_xor_sync(gmask, v1, o), w2 = __shfl_xor_sync(gmask, v2, o);
        const int j1 = __shfl_xor_sync(gmask, i1, o), j2 = __shfl_xor_sync(gmask, i2, o);
        // merge two (value desc, id asc) sorted pairs
        auto better = [](float a, int ia, float b, int ib) { return a > b || (a == b && ia < ib); };
        float r1, r2;
        int q1, q2;
        if (better(v1, i1, w1, j1)) {
          r1 = v1; q1 = i1;
          if (better(v2, i2, w1, j1)) { r2 = v2; q2 = i2; } else { r2 = w1; q2 = j1; }
        } else {
          r1 = w1; q1 = j1;
          if (better(v1, i1, w2, j2)) { r2 = v1; q2 = i1; } else { r2 = w2; q2 = j2; }
        }
        v1 = r1; i1 = q1; v2 = r2; i2 = q2;
      }
      float sum = 0.f;
      for (int e = sub; e < E; e += L) sum += expf(lg[e] - mx);
#pragma unroll
      for (int o = 1; o < L; o <<= 1) sum += __shfl_xor_sync(gmask, sum, o);
      if (!live) continue;
      const float inv = 1.f / sum;
      const long t = t0 + ti0;
      if (probs)
        for (int e = sub; e < E; e += L) probs[t * E + e] = expf(lg[e] - mx) * inv;
      if (sub == 0) {
        const float p1 = expf(v1 - mx) * inv, p2 = k == 2 ? expf(v2 - mx) * inv : 0.f;
        const float rn = renorm ? 1.f / (p1 + p2) : 1.f;
        idx[t * k] = i1;
        w[t * k] = p1 * rn;
        atomicAdd(&s_hist[i1], 1);
        if (k == 2) {
          idx[t * k + 1] = i2;
          w[t * k + 1] = p2 * rn;
          atomicAdd(&s_hist[i2], 1);
        }
      }
    }
  } else {
    for (int ti = threadIdx.x; ti < nt; ti += blockDim.x) {
      const long t = t0 + ti;
      finish_token(s_lg + (size_t)ti * ld, E, k, renorm, idx + t * k, w + t * k,
                   probs ? probs + t * E : nullptr, s_hist);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (s_hist[e]) atomicAdd(&hist[e], s_hist[e]);
}

// ---------------------------------------------------------------------------
// Fused router: logits[t, :] = x[t, :] . wg^T + bias, on the legacy mma.sync
// bf16 path (16 tokens x 8 experts per instruction; E <= 64 is far below the
// tcgen05 tile width, and the stage is bound by reading x from HBM).
// Each warp owns 16 tokens; lane (g = lane/4, t = lane%4) loads 16 contiguous
// bytes of rows g and g+8 per 32-wide k chunk.  The k order inside a chunk is
// permuted identically for A and B, which leaves the dot products unchanged.
// ---------------------------------------------------------------------------
constexpr int kRouterWarps = 8;
constexpr int kRouterTok = 16 * kRouterWarps;

__device__ __forceinline__ void mma_bf16_16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NT>
__global__ void __launch_bounds__(32 * kRouterWarps) router_gate_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
    const float* __restrict__ bias, int Tn, int d, int E, int k, int renorm,
    int32_t* __restrict__ idx, float* __restrict__ w, float* __restrict__ probs,
    int32_t* __restrict__ hist) {
  constexpr int EP = NT * 8 + 1;  // padded logit row (bank spread)
  __shared__ float s_log[kRouterWarps][16][EP];
  __shared__ int32_t s_hist[NT * 8];
  for (int e = threadIdx.x; e < NT * 8; e += blockDim.x) s_hist[e] = 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane >> 2, tq = lane & 3;
  const int tok0 = blockIdx.x * kRouterTok + warp * 16;
  const int r0 = tok0 + g, r1 = tok0 + g + 8;
  const bool v0 = r0 < Tn, v1 = r1 < Tn;
  const __nv_bfloat16* x0 = x + (size_t)(v0 ? r0 : 0) * d + 8 * tq;
  const __nv_bfloat16* x1 = x + (size_t)(v1 ? r1 : 0) * d + 8 * tq;
  const __nv_bfloat16* wrow[NT];
  bool wv[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int e = nt * 8 + g;
    wv[nt] = e < E;
    wrow[nt] = wg + (size_t)(wv[nt] ? e : 0) * d + 8 * tq;
  }
  float acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[nt][q] = 0.f;
  const uint4 zero = make_uint4(0, 0, 0, 0);
  if constexpr (NT <= 2) {
    constexpr int U = 4;  // k chunks in flight
    for (int kb = 0; kb < d; kb += 32 * U) {
      // all loads of the U chunks first (x rows and the router weights), then the MMAs
      uint4 xa[U], xb[U], bw[U][NT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kb + 32 * u;
        const bool in = kk < d;
        xa[u] = (v0 && in) ? ld_nc_v4(x0 + kk) : zero;
        xb[u] = (v1 && in) ? ld_nc_v4(x1 + kk) : zero;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bw[u][nt] = (wv[nt] && in) ? ld_v4(wrow[nt] + kk) : zero;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kb + 32 * u;
        if (kk >= d) break;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          mma_bf16_16816(acc[nt], xa[u].x, xb[u].x, xa[u].y, xb[u].y, bw[u][nt].x, bw[u][nt].y);
          mma_bf16_16816(acc[nt], xa[u].z, xb[u].z, xa[u].w, xb[u].w, bw[u][nt].z, bw[u][nt].w);
        }
      }
    }
  } else {
    // wide routers (E > 16): the x rows (HBM) stay U = 4 chunks ahead; the router weights
    // (L1/L2-resident, shared by every warp) are fetched per chunk, right before its MMAs
    constexpr int U = 4;
    for (int kb = 0; kb < d; kb += 32 * U) {
      uint4 xa[U], xb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kb + 32 * u;
        const bool in = kk < d;
        xa[u] = (v0 && in) ? ld_nc_v4(x0 + kk) : zero;
        xb[u] = (v1 && in) ? ld_nc_v4(x1 + kk) : zero;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kb + 32 * u;
        if (kk >= d) break;
        uint4 bw[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bw[nt] = wv[nt] ? ld_v4(wrow[nt] + kk) : zero;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          mma_bf16_16816(acc[nt], xa[u].x, xb[u].x, xa[u].y, xb[u].y, bw[nt].x, bw[nt].y);
          mma_bf16_16816(acc[nt], xa[u].z, xb[u].z, xa[u].w, xb[u].w, bw[nt].z, bw[nt].w);
        }
      }
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c0 = nt * 8 + 2 * tq;
    const float b0 = (bias && c0 < E) ? bias[c0] : 0.f;
    const float b1 = (bias && c0 + 1 < E) ? bias[c0 + 1] : 0.f;
    s_log[warp][g][c0] = acc[nt][0] + b0;
    s_log[warp][g][c0 + 1] = acc[nt][1] + b1;
    s_log[warp][g + 8][c0] = acc[nt][2] + b0;
    s_log[warp][g + 8][c0 + 1] = acc[nt][3] + b1;
  }
  __syncthreads();
  if (lane < 16) {
    const int t = tok0 + lane;
    if (t < Tn)
      finish_token(&s_log[warp][lane][0], E, k, renorm, idx + (size_t)t * k, w + (size_t)t * k,
                   probs ? probs + (size_t)t * E : nullptr, s_hist);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (s_hist[e]) atomicAdd(&hist[e], s_hist[e]);
}

// ---------------------------------------------------------------------------
// Wide routers (E > 16, d % 64 == 0): the register-direct kernel above has every warp
// re-read all of Wg (E x d x 2 bytes, 256 KB at E = 64, d = 2048 -- too big for L1), so
// the router weights dominate L2 traffic.  Here a block of 8 warps x 16 tokens streams
// x and Wg through a 4-stage cp.async ring of 64-column chunks shared by all its warps
// (A fragments by ldmatrix); the logits tile is then staged in the idle ring.
// ---------------------------------------------------------------------------
constexpr int kRgK = 64;                  // columns per stage
constexpr int kRgStages = 4;
constexpr int kRgXRow = kRgK + 8;         // bf16 per smem row (144 B: ldmatrix conflict-free)
template <int NT>
struct RgCfg {
  static constexpr int kXBytes = kRouterTok * kRgXRow * 2;
  static constexpr int kWBytes = NT * 8 * kRgXRow * 2;
  static constexpr int kStage = kXBytes + kWBytes;
  static constexpr int kSmem = kRgStages * kStage;
  static_assert(kRouterWarps * 16 * (NT * 8 + 1) * 4 <= kSmem, "logit tile fits the ring");
};
__device__ __forceinline__ void rg_cp16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(ok ? 16 : 0));
}
template <int NT>
__global__ void __launch_bounds__(32 * kRouterWarps, 2) router_gate_pipe(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
    const float* __restrict__ bias, int Tn, int d, int E, int k, int renorm,
    int32_t* __restrict__ idx, float* __restrict__ w, float* __restrict__ probs,
    int32_t* __restrict__ hist) {
  using C = RgCfg<NT>;
  extern __shared__ __align__(16) uint8_t rg_smem[];
  __shared__ int32_t s_hist[NT * 8];
  for (int e = threadIdx.x; e < NT * 8; e += blockDim.x) s_hist[e] = 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane >> 2, tq = lane & 3;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(rg_smem);
  const int nk = d / kRgK;
  const int nblocks = (Tn + kRouterTok - 1) / kRouterTok;
  for (int tb = blockIdx.x; tb < nblocks; tb += gridDim.x) {
    const long tok0 = (long)tb * kRouterTok;
    auto stage = [&](int buf, int kc) {
      const uint32_t sx = s0 + buf * C::kStage, sw = sx + C::kXBytes;
      for (int q = threadIdx.x; q < kRouterTok * 8; q += blockDim.x) {
        const int r = q >> 3, c = q & 7;
        const long t = tok0 + r;
        rg_cp16(sx + (r * kRgXRow + c * 8) * 2, x + (t < Tn ? t : 0) * d + kc * kRgK + c * 8,
                t < Tn);
      }
      for (int q = threadIdx.x; q < NT * 8 * 8; q += blockDim.x) {
        const int e = q >> 3, c = q & 7;
        rg_cp16(sw + (e * kRgXRow + c * 8) * 2,
                wg + (e < E ? e : 0) * (long)d + kc * kRgK + c * 8, e < E);
      }
      asm volatile("cp.async.commit_group;");
    };
#pragma unroll
    for (int i = 0; i < kRgStages - 1; ++i) {
      if (i < nk) stage(i, i);
      else asm volatile("cp.async.commit_group;");
    }
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[nt][q] = 0.f;
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc % kRgStages;
      asm volatile("cp.async.wait_group %0;" ::"n"(kRgStages - 2) : "memory");
      __syncthreads();
      {
        const int j = kc + kRgStages - 1;
        if (j < nk) stage(j % kRgStages, j);
        else asm volatile("cp.async.commit_group;");
      }
      const uint32_t sx = s0 + buf * C::kStage;
      const __nv_bfloat16* wsm =
          reinterpret_cast<const __nv_bfloat16*>(rg_smem + buf * C::kStage + C::kXBytes);
#pragma unroll
      for (int kk = 0; kk < kRgK / 16; ++kk) {
        uint32_t a0, a1, a2, a3;
        const uint32_t aaddr =
            sx + ((warp * 16 + (lane & 15)) * kRgXRow + kk * 16 + (lane >> 4) * 8) * 2;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                     : "r"(aaddr));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const __nv_bfloat16* wr = wsm + (nt * 8 + g) * kRgXRow + kk * 16 + 2 * tq;
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(wr);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(wr + 8);
          mma_bf16_16816(acc[nt], a0, a1, a2, a3, b0, b1);
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();   // ring idle: reuse it for the logits tile
    constexpr int EP = NT * 8 + 1;
    float* s_log = reinterpret_cast<float*>(rg_smem) + warp * 16 * EP;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c0 = nt * 8 + 2 * tq;
      const float b0 = (bias && c0 < E) ? bias[c0] : 0.f;
      const float b1 = (bias && c0 + 1 < E) ? bias[c0 + 1] : 0.f;
      s_log[g * EP + c0] = acc[nt][0] + b0;
      s_log[g * EP + c0 + 1] = acc[nt][1] + b1;
      s_log[(g + 8) * EP + c0] = acc[nt][2] + b0;
      s_log[(g + 8) * EP + c0 + 1] = acc[nt][3] + b1;
    }
    __syncwarp();
    if (lane < 16) {
      const long t = tok0 + warp * 16 + lane;
      if (t < Tn)
        finish_token(s_log + lane * EP, E, k, renorm, idx + t * k, w + t * k,
                     probs ? probs + t * E : nullptr, s_hist);
    }
    __syncthreads();   // logits tile consumed before the ring is refilled
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (s_hist[e]) atomicAdd(&hist[e], s_hist[e]);
}

// ---------------------------------------------------------------------------
// Streaming router for the common shape (E <= 16, d % 64 == 0, d <= 1024): one
// persistent CTA per SM owns a CONTIGUOUS token range, so x streams from HBM in order.
// Warp roles:
//   producer (1 lane)  moves each 16-token group (16 rows of d * 2 bytes) into a 4-stage
//                      shared-memory ring with cp.async.bulk (one copy per row into
//                      16-byte-padded rows: conflict-free ldmatrix), completing on an
//                      mbarrier;
//   4 MMA warps        split the d columns (d / 4 each) and run mma.sync against Wg held
//                      in shared memory; each writes its 16 x 16 partial logits to its
//                      slot of one of 12 rotating tiles (tile_full: 4 arrivals);
//   6 finisher warps   take the groups round-robin: sum the 4 slots in a fixed order
//                      (deterministic and independent of the token's batch position)
//                      + bias, softmax / top-k with one lane per token, then release the
//                      tile (tile_empty).
// The register-direct kernel below needs 2 waves of 16-token warps at 64K tokens, each
// warp latency-bound on 4 KB in flight.
// ---------------------------------------------------------------------------
// warp / ring shape of the streaming router: (MMA warps, finisher warps, stages, tiles) =
// (4, 6, 4, 12); measured against (8, 6, 4, 6), (4, 8, 4, 12), (8, 4, 4, 6), (4, 6, 3, 12):
// all within 28.8-29.9 us at cfg2 -- the kernel is bound by its fixed per-launch costs
#ifndef LZ_GS_MMA
#define LZ_GS_MMA 4
#define LZ_GS_FIN 6
#define LZ_GS_STAGES 4
#define LZ_GS_TILES 12
#endif
constexpr int kGsMma = LZ_GS_MMA;         // MMA (column-split) warps
constexpr int kGsFin = LZ_GS_FIN;         // finisher warps
constexpr int kGsStages = LZ_GS_STAGES;   // x ring depth
constexpr int kGsTiles = LZ_GS_TILES;     // partial-logit tiles
constexpr int kGsEP = 17;         // padded partial row (16 experts + 1)
constexpr int kGsThreads = 32 * (kGsMma + kGsFin + 1);
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void gs_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void gs_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int NT>
__global__ void __launch_bounds__(kGsThreads, 1) router_gate_stream(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
    const float* __restrict__ bias, int Tn, int d, int E, int k, int renorm,
    int32_t* __restrict__ idx, float* __restrict__ w, float* __restrict__ probs,
    int32_t* __restrict__ hist, int32_t* __restrict__ hist_ws) {
  extern __shared__ __align__(128) uint8_t gs_smem[];
  __shared__ __align__(8) uint64_t full_bar[kGsStages], empty_bar[kGsStages];
  __shared__ __align__(8) uint64_t tfull_bar[kGsTiles], tempty_bar[kGsTiles];
  __shared__ int32_t s_hist[16];
  pdl_launch_dependents();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rowb = (d + 8) * 2;                    // padded smem row, bytes
  uint8_t* ring = gs_smem;                         // [stages][16][d + 8] bf16
  uint8_t* wsm = ring + kGsStages * 16 * rowb;     // [16][d + 8] bf16
  float* part = reinterpret_cast<float*>(wsm + 16 * rowb);  // [tiles][kGsMma][16][kGsEP]
  const int ng = (Tn + 15) / 16;
  const int g_begin = (int)((long)ng * blockIdx.x / gridDim.x);
  const int g_end = (int)((long)ng * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x < 16) s_hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGsStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full_bar[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty_bar[i])),
                   "r"(kGsMma));
    }
    for (int i = 0; i < kGsTiles; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&tfull_bar[i])),
                   "r"(kGsMma));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tempty_bar[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // producer: lane r issues row r's copy of a 16-token group (16 bulk copies per instruction)
  auto issue = [&](int gi, int i) {
    const int st = i % kGsStages;
    const long t0 = (long)gi * 16;
    const int nv = (int)min(16L, (long)Tn - t0);
    const uint32_t fb = smem_u32(&full_bar[st]);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                   "r"((uint32_t)(nv * d * 2))
                   : "memory");
    __syncwarp();
    if (lane < nv)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(smem_u32(ring + st * 16 * rowb) + lane * rowb),
          "l"(x + (t0 + lane) * d), "r"(d * 2), "r"(fb)
          : "memory");
  };
  const bool producer = warp == kGsMma + kGsFin;
  {
    // router weights -> smem (rows >= E zero), every thread's loads in flight at once
    constexpr int kPer = (16 * 1024 / 8 + kGsThreads - 1) / kGsThreads;   // d <= 1024
    const int nq = 16 * (d / 8);
    uint4 v[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int q = threadIdx.x + j * kGsThreads;
      const int e = q / (d / 8), c = q % (d / 8);
      v[j] = (q < nq && e < E) ? ld_v4(wg + (long)e * d + c * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int q = threadIdx.x + j * kGsThreads;
      if (q < nq)
        *reinterpret_cast<uint4*>(wsm + (q / (d / 8)) * rowb + (q % (d / 8)) * 16) = v[j];
    }
  }
  __syncthreads();
  if (producer) {
    // the barrier init and the router-weight staging above overlap the predecessor's tail
    // (PDL; no kernel of the step writes wg); x and every output only after the wait
    pdl_wait();
    for (int i = 0; i < kGsStages && g_begin + i < g_end; ++i) issue(g_begin + i, i);
    for (int gi = g_begin + kGsStages, i = kGsStages; gi < g_end; ++gi, ++i) {
      gs_wait(&empty_bar[i % kGsStages], ((i / kGsStages) - 1) & 1);
      issue(gi, i);
    }
  } else if (warp < kGsMma) {
    // ===== MMA warps: columns [warp * d / 4, +d / 4) =====
    const int g = lane >> 2, tq = lane & 3;
    const int cw = d / kGsMma;
    const int c_base = warp * cw;
    for (int gi = g_begin, i = 0; gi < g_end; ++gi, ++i) {
      const int st = i % kGsStages;
      gs_wait(&full_bar[st], (i / kGsStages) & 1);
      float acc[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[nt][q] = 0.f;
      const uint32_t sx = smem_u32(ring + st * 16 * rowb);
#pragma unroll 4
      for (int kk = 0; kk < cw; kk += 16) {
        const int c = c_base + kk;
        uint32_t a0, a1, a2, a3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                     : "r"(sx + (lane & 15) * rowb + (c + (lane >> 4) * 8) * 2));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint8_t* wr = wsm + (nt * 8 + g) * rowb + (c + 2 * tq) * 2;
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(wr);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(wr + 16);
          mma_bf16_16816(acc[nt], a0, a1, a2, a3, b0, b1);
        }
      }
      __syncwarp();
      if (lane == 0) gs_arrive(&empty_bar[st]);
      const int tile = i % kGsTiles;
      if (i >= kGsTiles) gs_wait(&tempty_bar[tile], ((i / kGsTiles) - 1) & 1);
      float* pw = part + ((tile * kGsMma + warp) * 16) * kGsEP;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c0 = nt * 8 + 2 * tq;
        pw[g * kGsEP + c0] = acc[nt][0];
        pw[g * kGsEP + c0 + 1] = acc[nt][1];
        pw[(g + 8) * kGsEP + c0] = acc[nt][2];
        pw[(g + 8) * kGsEP + c0 + 1] = acc[nt][3];
      }
      __syncwarp();
      if (lane == 0) gs_arrive(&tfull_bar[tile]);
    }
  } else {
    // ===== finisher warps: groups f, f + kGsFin, ... =====
    const int f = warp - kGsMma;
    for (int i = f; g_begin + i < g_end; i += kGsFin) {
      const int tile = i % kGsTiles;
      gs_wait(&tfull_bar[tile], (i / kGsTiles) & 1);
      const long t = (long)(g_begin + i) * 16 + lane;
      if (lane < 16 && t < Tn) {
        float* lg = part + ((tile * kGsMma) * 16 + lane) * kGsEP;  // MMA warp 0's slot
        for (int e = 0; e < E; ++e) {
          float v = lg[e];
#pragma unroll
          for (int ww = 1; ww < kGsMma; ++ww) v += lg[ww * 16 * kGsEP + e];
          lg[e] = v + (bias ? __ldg(bias + e) : 0.f);
        }
        finish_token(lg, E, k, renorm, idx + t * k, w + t * k, probs ? probs + t * E : nullptr,
                     s_hist);
      }
      __syncwarp();
      if (lane == 0) gs_arrive(&tempty_bar[tile]);
    }
  }
  __syncthreads();
  // histogram without a memset in front: every CTA stores its 16 counts into its row of a
  // per-launch workspace slot; the last CTA to arrive (ticket) sums the rows in a fixed
  // order into hist and resets the ticket for the slot's next use
  int32_t* ticket = hist_ws;
  int32_t* rows = hist_ws + 32;
  if (threadIdx.x < 16) rows[blockIdx.x * 16 + threadIdx.x] = s_hist[threadIdx.x];
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    __shared__ int32_t s_sum[kGsThreads / 16][16];
    const int e = threadIdx.x & 15, j = threadIdx.x >> 4;   // 22 row groups x 16 experts
    int32_t v = 0;
    for (int b = j; b < (int)gridDim.x; b += kGsThreads / 16)
      v += *reinterpret_cast<volatile int32_t*>(rows + b * 16 + e);
    s_sum[j][e] = v;
    __syncthreads();
    if (threadIdx.x < E) {
      int32_t tot = 0;
      for (int jj = 0; jj < kGsThreads / 16; ++jj) tot += s_sum[jj][threadIdx.x];
      hist[threadIdx.x] = tot;
    }
    if (threadIdx.x == 0) *ticket = 0;
  }
}
// per-launch histogram workspaces of the streaming router (ticket + one 16-count row per
// CTA), a rolling pool: a slot is reused only 256 launches later (also by every replay of a
// captured graph, whose launch keeps its slot); the ticket self-resets
constexpr int kGsWsSlots = 256, kGsWsInts = 32 + 256 * 16;
__device__ int32_t g_gate_ws[kGsWsSlots][kGsWsInts];
__host__ __device__ constexpr size_t gs_smem_bytes(int d) {
  return (size_t)(kGsStages + 1) * 16 * (d + 8) * 2 +
         (size_t)kGsTiles * kGsMma * 16 * kGsEP * sizeof(float);
}

// Gate backward alone (thread per token): dlogits from probs, idx and the combine
// backward's dw -- the values lz_dispatch_bwd also produces (same gate_bwd_coefs), available
// right after the combine backward, so the router weight gradient can start there.
__global__ void __launch_bounds__(256) gate_bwd_kernel(const float* __restrict__ probs,
                                                       const int32_t* __restrict__ idx,
                                                       const float* __restrict__ dw, int Tn,
                                                       int E, int k, int renorm,
                                                       float* __restrict__ dlogits) {
  pdl_prologue();
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Tn) return;
  int ids[LZ_MAX_TOPK];
  float ps[LZ_MAX_TOPK], g[LZ_MAX_TOPK];
#pragma unroll
  for (int s = 0; s < LZ_MAX_TOPK; ++s) {
    ids[s] = -1;
    ps[s] = g[s] = 0.f;
    if (s < k) {
      ids[s] = __ldg(idx + t * k + s);
      g[s] = __ldg(dw + t * k + s);
      ps[s] = __ldg(probs + t * E + ids[s]);
    }
  }
  const float dot = gate_bwd_coefs(k, renorm, ps, g);
  const float* pr = probs + t * E;
  float* out = dlogits + t * E;
  if (E % 4 == 0) {
    for (int e = 0; e < E; e += 4) {
      const float4 p4 = __ldg(reinterpret_cast<const float4*>(pr + e));
      *reinterpret_cast<float4*>(out + e) =
          make_float4(gate_bwd_dl(p4.x, e, dot, ids, g), gate_bwd_dl(p4.y, e + 1, dot, ids, g),
                      gate_bwd_dl(p4.z, e + 2, dot, ids, g), gate_bwd_dl(p4.w, e + 3, dot, ids, g));
    }
  } else {
    for (int e = 0; e < E; ++e) out[e] = gate_bwd_dl(__ldg(pr + e), e, dot, ids, g);
  }
}

}  // namespace lz

using namespace lz;

extern "C" lz_status lz_gate_bwd(const float* probs, const int32_t* idx, const float* dw, int Tn,
                                 int E, int k, int renorm, float* dlogits, void* stream) {
  if (Tn < 0 || E < 1 || E > LZ_MAX_EXPERTS || k < 1 || k > LZ_MAX_TOPK || k > E) return LZ_ERR_ARG;
  if (Tn == 0) return LZ_OK;
  if (!probs || !idx || !dw || !dlogits) return LZ_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(probs) | reinterpret_cast<uintptr_t>(dlogits)) % 16)
    return LZ_ERR_ARG;
  return lzh::launch(gate_bwd_kernel, dim3((Tn + 255) / 256), dim3(256), 0, (cudaStream_t)stream,
                     1, probs, idx, dw, Tn, E, k, renorm, dlogits);
}

extern "C" lz_status lz_gate_topk(const float* logits, int Tn, int E, int k, int renorm,
                                  int32_t* idx, float* w, float* probs, int32_t* hist,
                                  void* stream) {
  if (Tn < 0 || E < 1 || E > LZ_MAX_EXPERTS || k < 1 || k > LZ_MAX_TOPK || k > E || !hist)
    return LZ_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(hist, 0, sizeof(int32_t) * E, s) != cudaSuccess) return lzh::check_launch();
  if (Tn == 0) return LZ_OK;
  if (!logits || !idx || !w) return LZ_ERR_ARG;
  int tpb = 16384 / (E + 1);
  tpb = tpb > 256 ? 256 : (tpb < 1 ? 1 : tpb);
  const size_t smem = sizeof(float) * (size_t)tpb * (E + 1) + sizeof(int32_t) * E;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(gate_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             80 * 1024) != cudaSuccess)
      return lzh::check_launch();
    attr = true;
  }
  gate_topk_kernel<<<(int)((Tn + tpb - 1) / tpb), 256, smem, s>>>(logits, Tn, E, k, renorm, tpb,
                                                                  idx, w, probs, hist);
  return lzh::check_launch();
}

extern "C" lz_status lz_router_gate(const void* x, const void* wg, const float* bias, int Tn,
                                    int d, int E, int k, int renorm, int32_t* idx, float* w,
                                    float* probs, int32_t* hist, void* stream) {
  if (Tn < 0 || d < 32 || d % 32 || E < 1 || E > 64 || k < 1 || k > LZ_MAX_TOPK || k > E ||
      !hist)
    return LZ_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool stream_kernel = E <= 16 && d % 64 == 0 && d <= 1024 && Tn > 0;
  // the streaming kernel writes the histogram itself (no memset node in front of it)
  if (!stream_kernel && cudaMemsetAsync(hist, 0, sizeof(int32_t) * E, s) != cudaSuccess)
    return lzh::check_launch();
  if (Tn == 0) return LZ_OK;
  if (!x || !wg || !idx || !w) return LZ_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(wg)) % 16) return LZ_ERR_ARG;
  const int grid = (Tn + kRouterTok - 1) / kRouterTok;
  const auto* xb = (const __nv_bfloat16*)x;
  const auto* wb = (const __nv_bfloat16*)wg;
  const int NT = (E + 7) / 8;
  if (stream_kernel) {
    // streaming kernel: one persistent CTA per SM over a contiguous token range (for
    // every Tn, so a token's logits never depend on the batch it came in)
    const size_t smem = gs_smem_bytes(d);
    const int ngroups = (Tn + 15) / 16;
    int sgrid = ngroups < lzh::num_sms() ? ngroups : lzh::num_sms();
    if (sgrid > 256) sgrid = 256;
    static int32_t* ws_base = nullptr;
    static unsigned ws_next = 0;
    if (!ws_base) {
      void* ptr = nullptr;
      if (cudaGetSymbolAddress(&ptr, g_gate_ws) != cudaSuccess) return lzh::check_launch();
      ws_base = (int32_t*)ptr;
    }
    int32_t* hist_ws = ws_base + (size_t)(ws_next++ % kGsWsSlots) * kGsWsInts;
#define LZ_ROUTER_STREAM(n)                                                                 \
  case n: {                                                                                 \
    static bool attr = false;                                                               \
    if (!attr) {                                                                            \
      if (cudaFuncSetAttribute(router_gate_stream<n>,                                       \
                               cudaFuncAttributeMaxDynamicSharedMemorySize,                 \
                               (int)gs_smem_bytes(1024)) != cudaSuccess)                    \
        return lzh::check_launch();                                                         \
      attr = true;                                                                          \
    }                                                                                       \
    lzh::launch(router_gate_stream<n>, dim3(sgrid), dim3(kGsThreads), smem, s, 1, xb, wb,  \
                bias, Tn, d, E, k, renorm, idx, w, probs, hist, hist_ws);                   \
    break;                                                                                  \
  }
    switch (NT) {
      LZ_ROUTER_STREAM(1)
      LZ_ROUTER_STREAM(2)
      default:
        return LZ_ERR_UNSUPPORTED;
    }
#undef LZ_ROUTER_STREAM
    return lzh::check_launch();
  }
  if (NT > 2 && d % kRgK == 0) {
    // wide router: the block-shared pipelined kernel (persistent, 2 blocks per SM)
    const int pgrid = grid < 2 * lzh::num_sms() ? grid : 2 * lzh::num_sms();
#define LZ_ROUTER_PIPE(n)                                                                    \
  case n: {                                                                                  \
    static bool attr = false;                                                                \
    if (!attr) {                                                                             \
      if (cudaFuncSetAttribute(router_gate_pipe<n>,                                          \
                               cudaFuncAttributeMaxDynamicSharedMemorySize,                  \
                               RgCfg<n>::kSmem) != cudaSuccess)                              \
        return lzh::check_launch();                                                          \
      attr = true;                                                                           \
    }                                                                                        \
    router_gate_pipe<n><<<pgrid, 32 * kRouterWarps, RgCfg<n>::kSmem, s>>>(                   \
        xb, wb, bias, Tn, d, E, k, renorm, idx, w, probs, hist);                             \
    break;                                                                                   \
  }
    switch (NT) {
      LZ_ROUTER_PIPE(3)
      LZ_ROUTER_PIPE(4)
      LZ_ROUTER_PIPE(5)
      LZ_ROUTER_PIPE(6)
      LZ_ROUTER_PIPE(7)
      LZ_ROUTER_PIPE(8)
      default:
        return LZ_ERR_UNSUPPORTED;
    }
#undef LZ_ROUTER_PIPE
    return lzh::check_launch();
  }
#define LZ_ROUTER_CASE(n)                                                                    \
  case n:                                                                                    \
    router_gate_kernel<n><<<grid, 32 * kRouterWarps, 0, s>>>(xb, wb, bias, Tn, d, E, k,       \
                                                             renorm, idx, w, probs, hist);   \
    break;
  switch (NT) {
    LZ_ROUTER_CASE(1)
    LZ_ROUTER_CASE(2)
    LZ_ROUTER_CASE(3)
    LZ_ROUTER_CASE(4)
    LZ_ROUTER_CASE(5)
    LZ_ROUTER_CASE(6)
    LZ_ROUTER_CASE(7)
    LZ_ROUTER_CASE(8)
    default:
      return LZ_ERR_UNSUPPORTED;
  }
#undef LZ_ROUTER_CASE
  return lzh::check_launch();
}
