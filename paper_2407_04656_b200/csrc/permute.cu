// permute.cu -- K3 pack, K7 combine, K8 backward permutes, router weight grad.
//
// All of these are HBM-bound row movers: one warp per token row, 16-byte
// vectorised coalesced loads/stores, 4 vectors in flight per lane, streaming
// (L1::no_allocate) loads for read-once activations.  Reference semantics:
//   pack     Alg. 1 reshuffle: token rows go to the send/receive
//            slot the planner assigned (dispatch.py:199-237 gives the index only)
//   combine  PAPER.md:99 weighted sum of the k expert outputs (fixed s order)
#include "common.cuh"

namespace lz {

constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / 32;
constexpr int kVec = 4;  // uint4 per lane in flight

__device__ __forceinline__ void zero_pad_rows(void* out, int d, int E, const int32_t* recv_m,
                                              const int32_t* recv_off, long item, long n_items,
                                              int lane) {
  // item enumerates (expert, pad row) pairs; pad rows are [off[e]+m[e], off[e+1])
  (void)n_items;
  const int nch = d / 8;
  for (int e = 0; e < E; ++e) {
    const long start = (long)recv_off[e] + recv_m[e];
    const long cnt = (long)recv_off[e + 1] - start;
    if (item < cnt) {
      uint4* dst = reinterpret_cast<uint4*>(out) + (start + item) * nch;
      for (int c = lane; c < nch; c += 32) st_v4(dst + c, make_uint4(0, 0, 0, 0));
      return;
    }
    item -= cnt;
  }
}

// Row base for assignment slot s of the current token: a peer's symmetric buffer
// (NVLink P2P, `peers[rank]`) when `peers` is given, else the local buffer.
__device__ __forceinline__ uint4* row_base(uint4* local, const unsigned long long* peers,
                                           int my_rk, int s) {
  if (!peers) return local;
  const int r = __shfl_sync(0xffffffffu, my_rk, s);
  return reinterpret_cast<uint4*>(peers[r]);
}

__global__ void __launch_bounds__(kRowThreads) pack_kernel(
    const uint4* __restrict__ x, int Tn, int d, int k, const int32_t* __restrict__ row,
    const int32_t* __restrict__ prank, const unsigned long long* __restrict__ peers,
    uint4* __restrict__ out, int E, const int32_t* __restrict__ recv_m,
    const int32_t* __restrict__ recv_off, long n_pad_items) {
  const int lane = threadIdx.x % 32;
  const long gw = (long)blockIdx.x * kRowWarps + threadIdx.x / 32;
  const long nw = (long)gridDim.x * kRowWarps;
  const int nch = d / 8;
  for (long t = gw; t < Tn + n_pad_items; t += nw) {
    if (t >= Tn) {
      zero_pad_rows(out, d, E, recv_m, recv_off, t - Tn, n_pad_items, lane);
      continue;
    }
    const int my_row = lane < k ? __ldg(row + t * k + lane) : 0;
    const int my_rk = (peers && lane < k) ? __ldg(prank + t * k + lane) : 0;
    const uint4* src = x + t * nch;
    for (int c0 = lane; c0 < nch; c0 += 32 * kVec) {
      uint4 v[kVec];
#pragma unroll
      for (int u = 0; u < kVec; ++u)
        if (c0 + 32 * u < nch) v[u] = ld_nc_v4(src + c0 + 32 * u);
      for (int s = 0; s < k; ++s) {
        const long r = __shfl_sync(0xffffffffu, my_row, s);
        uint4* dst = row_base(out, peers, my_rk, s) + r * nch;
#pragma unroll
        for (int u = 0; u < kVec; ++u)
          if (c0 + 32 * u < nch) st_v4(dst + c0 + 32 * u, v[u]);
      }
    }
  }
}

__global__ void __launch_bounds__(kRowThreads) combine_kernel(
    const uint4* __restrict__ y, const int32_t* __restrict__ row, const int32_t* __restrict__ prank,
    const unsigned long long* __restrict__ peers, const float* __restrict__ w, int Tn, int d, int k,
    uint4* __restrict__ out) {
  const int lane = threadIdx.x % 32;
  const long gw = (long)blockIdx.x * kRowWarps + threadIdx.x / 32;
  const long nw = (long)gridDim.x * kRowWarps;
  const int nch = d / 8;
  for (long t = gw; t < Tn; t += nw) {
    const int my_row = lane < k ? __ldg(row + t * k + lane) : 0;
    const float my_w = lane < k ? __ldg(w + t * k + lane) : 0.f;
    const int my_rk = (peers && lane < k) ? __ldg(prank + t * k + lane) : 0;
    for (int c0 = lane; c0 < nch; c0 += 32 * kVec) {
      float acc[kVec][8];
#pragma unroll
      for (int u = 0; u < kVec; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[u][q] = 0.f;
      for (int s = 0; s < k; ++s) {
        const long r = __shfl_sync(0xffffffffu, my_row, s);
        const float ws = __shfl_sync(0xffffffffu, my_w, s);
        const uint4* src = row_base(const_cast<uint4*>(y), peers, my_rk, s) + r * nch;
        uint4 v[kVec];
#pragma unroll
        for (int u = 0; u < kVec; ++u)
          if (c0 + 32 * u < nch) v[u] = ld_nc_v4(src + c0 + 32 * u);
#pragma unroll
        for (int u = 0; u < kVec; ++u) {
          if (c0 + 32 * u < nch) {
            float f[8];
            bf16x8_to_f32(v[u], f);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[u][q] = fmaf(ws, f[q], acc[u][q]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kVec; ++u)
        if (c0 + 32 * u < nch) st_v4(out + t * nch + c0 + 32 * u, f32_to_bf16x8(acc[u]));
    }
  }
}

__global__ void __launch_bounds__(kRowThreads) combine_bwd_kernel(
    const uint4* __restrict__ dout, const uint4* __restrict__ y, const int32_t* __restrict__ row,
    const int32_t* __restrict__ prank, const unsigned long long* __restrict__ peers_y,
    const unsigned long long* __restrict__ peers_dy,
    const float* __restrict__ w, int Tn, int d, int k, uint4* __restrict__ dy,
    float* __restrict__ dw, int E, const int32_t* __restrict__ recv_m,
    const int32_t* __restrict__ recv_off, long n_pad_items) {
  const int lane = threadIdx.x % 32;
  const long gw = (long)blockIdx.x * kRowWarps + threadIdx.x / 32;
  const long nw = (long)gridDim.x * kRowWarps;
  const int nch = d / 8;
  for (long t = gw; t < Tn + n_pad_items; t += nw) {
    if (t >= Tn) {
      zero_pad_rows(dy, d, E, recv_m, recv_off, t - Tn, n_pad_items, lane);
      continue;
    }
    const int my_row = lane < k ? __ldg(row + t * k + lane) : 0;
    const float my_w = lane < k ? __ldg(w + t * k + lane) : 0.f;
    const int my_rk = (peers_y && lane < k) ? __ldg(prank + t * k + lane) : 0;
    float dot[LZ_MAX_TOPK];
#pragma unroll
    for (int s = 0; s < LZ_MAX_TOPK; ++s) dot[s] = 0.f;
    for (int c0 = lane; c0 < nch; c0 += 32 * kVec) {
      float g[kVec][8];
#pragma unroll
      for (int u = 0; u < kVec; ++u)
        if (c0 + 32 * u < nch) bf16x8_to_f32(ld_nc_v4(dout + t * nch + c0 + 32 * u), g[u]);
#pragma unroll
      for (int s = 0; s < LZ_MAX_TOPK; ++s) {
        if (s >= k) break;
        const long r = __shfl_sync(0xffffffffu, my_row, s);
        const float ws = __shfl_sync(0xffffffffu, my_w, s);
        const uint4* ys = row_base(const_cast<uint4*>(y), peers_y, my_rk, s) + r * nch;
        uint4* dys = row_base(dy, peers_dy, my_rk, s) + r * nch;
        uint4 v[kVec];
#pragma unroll
        for (int u = 0; u < kVec; ++u)
          if (c0 + 32 * u < nch) v[u] = ld_nc_v4(ys + c0 + 32 * u);
#pragma unroll
        for (int u = 0; u < kVec; ++u) {
          if (c0 + 32 * u < nch) {
            float f[8], o[8];
            bf16x8_to_f32(v[u], f);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              dot[s] = fmaf(g[u][q], f[q], dot[s]);
              o[q] = ws * g[u][q];
            }
            st_v4(dys + c0 + 32 * u, f32_to_bf16x8(o));
          }
        }
      }
    }
#pragma unroll
    for (int s = 0; s < LZ_MAX_TOPK; ++s) {
      if (s >= k) break;
      const float tot = warp_sum(dot[s]);
      if (lane == 0) dw[t * k + s] = tot;
    }
  }
}

// Gate backward (softmax + top-k (+renorm)) and dispatch backward.  A warp owns 16
// tokens.  Phase A computes their dlogits (lane = expert) into smem; phase B sweeps the
// row 64 columns at a time as a register-tiled 16 x 64 x E product (lane = 4 tokens x 8
// columns, one 16-byte wg load feeds 32 FMAs) plus the gathered expert rows
// sum_s dxe[row(t, s)], stored with 128-byte coalesced rows.
constexpr int kDT = 16;
__global__ void __launch_bounds__(kRowThreads) dispatch_bwd_kernel(
    const uint4* __restrict__ dxe, const int32_t* __restrict__ row,
    const int32_t* __restrict__ prank, const unsigned long long* __restrict__ peers, int Tn, int d,
    int k, const float* __restrict__ probs, const int32_t* __restrict__ idx,
    const float* __restrict__ dwv, const __nv_bfloat16* __restrict__ wg, int E, int renorm,
    uint4* __restrict__ dx, float* __restrict__ dlogits) {
  __shared__ __align__(16) float s_dl[kRowWarps][64][kDT];        // [expert][token]
  __shared__ long long s_src[kRowWarps][kDT][LZ_MAX_TOPK];        // row base per (token, s)
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const long gw = (long)blockIdx.x * kRowWarps + warp;
  const long nw = (long)gridDim.x * kRowWarps;
  const int nch = d / 8;
  const int tq = lane >> 3;        // token quad: tokens 4*tq .. 4*tq+3
  const int cq = lane & 7;         // 16-byte column chunk inside the 64-column pass
  for (long t0 = gw * kDT; t0 < Tn; t0 += nw * kDT) {
    // ---- phase A: dlogits of the 16 tokens ------------------------------------
    for (int ti = 0; ti < kDT; ++ti) {
      const long t = t0 + ti;
      if (t >= Tn) {
        s_dl[warp][lane][ti] = 0.f;
        s_dl[warp][lane + 32][ti] = 0.f;
        continue;
      }
      const int my_row = lane < k ? __ldg(row + t * k + lane) : 0;
      const int my_idx = lane < k ? __ldg(idx + t * k + lane) : -1;
      const float my_dw = lane < k ? __ldg(dwv + t * k + lane) : 0.f;
      const int my_rk = (peers && lane < k) ? __ldg(prank + t * k + lane) : 0;
      if (lane < k) {
        const uint4* base = peers ? reinterpret_cast<const uint4*>(peers[my_rk]) : dxe;
        s_src[warp][ti][lane] = (long long)(base + (long)my_row * nch);
      }
      float p[2] = {0.f, 0.f}, dp[2] = {0.f, 0.f};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = lane + 32 * h;
        if (e < E) p[h] = __ldg(probs + t * E + e);
      }
      float S = 0.f, sum_dw_w = 0.f;
      if (renorm) {
        for (int s2 = 0; s2 < k; ++s2) {
          const int es = __shfl_sync(0xffffffffu, my_idx, s2);
          S += __ldg(probs + t * E + es);
        }
        for (int s2 = 0; s2 < k; ++s2) {
          const int es = __shfl_sync(0xffffffffu, my_idx, s2);
          const float dws = __shfl_sync(0xffffffffu, my_dw, s2);
          sum_dw_w += dws * (__ldg(probs + t * E + es) / S);
        }
      }
      for (int s2 = 0; s2 < k; ++s2) {
        const int es = __shfl_sync(0xffffffffu, my_idx, s2);
        const float dws = __shfl_sync(0xffffffffu, my_dw, s2);
        const float g = renorm ? (dws - sum_dw_w) / S : dws;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (es == lane + 32 * h) dp[h] += g;
      }
      const float pdp = warp_sum(p[0] * dp[0] + p[1] * dp[1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = lane + 32 * h;
        const float dl = p[h] * (dp[h] - pdp);
        s_dl[warp][e][ti] = dl;
        if (e < E) dlogits[t * E + e] = dl;
      }
    }
    __syncwarp();
    const int nt = (int)min((long)kDT, Tn - t0);
    // ---- phase B: dx rows, 64 columns per pass -----------------------------------
    for (int c = cq; c < nch; c += 8) {
      // issue the gathered expert-row loads first (k <= 2 fast path); the E-long FMA
      // loop below hides their latency
      uint4 pre[4][2];
      const bool fast = k <= 2;
      if (fast) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ti = 4 * tq + i;
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2)
            pre[i][s2] = (ti < nt && s2 < k)
                             ? ld_nc_v4(reinterpret_cast<const uint4*>(s_src[warp][ti][s2]) + c)
                             : make_uint4(0, 0, 0, 0);
        }
      }
      float acc[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[i][q] = 0.f;
      if (wg) {
        for (int e = 0; e < E; ++e) {
          float w[8];
          bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(wg + (long)e * d) + c), w);
          const float4 dl4 = *reinterpret_cast<const float4*>(&s_dl[warp][e][4 * tq]);
          const float dlv[4] = {dl4.x, dl4.y, dl4.z, dl4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[i][q] = fmaf(dlv[i], w[q], acc[i][q]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ti = 4 * tq + i;
        if (ti < nt) {
          if (fast) {
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              float f[8];
              bf16x8_to_f32(pre[i][s2], f);
#pragma unroll
              for (int q = 0; q < 8; ++q) acc[i][q] += f[q];
            }
          } else {
            for (int s2 = 0; s2 < k; ++s2) {
              const uint4* src = reinterpret_cast<const uint4*>(s_src[warp][ti][s2]);
              float f[8];
              bf16x8_to_f32(ld_nc_v4(src + c), f);
#pragma unroll
              for (int q = 0; q < 8; ++q) acc[i][q] += f[q];
            }
          }
          st_v4(dx + (t0 + ti) * nch + c, f32_to_bf16x8(acc[i]));
        }
      }
    }
    __syncwarp();
  }
}

// dwg partials: block (bx, by, bz) reduces its token stripe for columns
// [by*1024, +1024) and experts [bz*16, +16); thread owns 4 columns x 16 experts.
constexpr int kWgE = 16;
constexpr int kWgTokTile = 64;
__global__ void __launch_bounds__(256, 2) router_wgrad_partial(const float* __restrict__ dlog,
                                                            const __nv_bfloat16* __restrict__ x,
                                                            int Tn, int d, int E,
                                                            float* __restrict__ part,
                                                            float* __restrict__ part_bias) {
  __shared__ float s_dl[kWgTokTile][kWgE];
  const int nblk = gridDim.x;
  const int col = blockIdx.y * 1024 + threadIdx.x * 4;
  const int e0 = blockIdx.z * kWgE;
  float acc[kWgE][4];
#pragma unroll
  for (int e = 0; e < kWgE; ++e)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[e][q] = 0.f;
  float bacc = 0.f;
  const long per = (Tn + nblk - 1) / nblk;
  const long t_begin = (long)blockIdx.x * per;
  const long t_end = min((long)Tn, t_begin + per);
  for (long tt = t_begin; tt < t_end; tt += kWgTokTile) {
    __syncthreads();
    for (int q = threadIdx.x; q < kWgTokTile * kWgE; q += blockDim.x) {
      const int ti = q / kWgE, ei = q % kWgE;
      const long t = tt + ti;
      s_dl[ti][ei] = (t < t_end && e0 + ei < E) ? dlog[t * E + e0 + ei] : 0.f;
    }
    __syncthreads();
    const int nt = (int)min((long)kWgTokTile, t_end - tt);
    if (blockIdx.y == 0 && threadIdx.x < kWgE)
      for (int ti = 0; ti < nt; ++ti) bacc += s_dl[ti][threadIdx.x];
    if (col < d) {
      int ti = 0;
      for (; ti + 8 <= nt; ti += 8) {
        uint2 raw[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          raw[u] = __ldg(reinterpret_cast<const uint2*>(x + (tt + ti + u) * d + col));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float x0 = __uint_as_float(raw[u].x << 16);
          const float x1 = __uint_as_float(raw[u].x & 0xffff0000u);
          const float x2 = __uint_as_float(raw[u].y << 16);
          const float x3 = __uint_as_float(raw[u].y & 0xffff0000u);
#pragma unroll
          for (int e = 0; e < kWgE; ++e) {
            const float g = s_dl[ti + u][e];
            acc[e][0] = fmaf(g, x0, acc[e][0]);
            acc[e][1] = fmaf(g, x1, acc[e][1]);
            acc[e][2] = fmaf(g, x2, acc[e][2]);
            acc[e][3] = fmaf(g, x3, acc[e][3]);
          }
        }
      }
      for (; ti < nt; ++ti) {
        const uint2 raw = __ldg(reinterpret_cast<const uint2*>(x + (tt + ti) * d + col));
        const float x0 = __uint_as_float(raw.x << 16), x1 = __uint_as_float(raw.x & 0xffff0000u);
        const float x2 = __uint_as_float(raw.y << 16), x3 = __uint_as_float(raw.y & 0xffff0000u);
#pragma unroll
        for (int e = 0; e < kWgE; ++e) {
          const float g = s_dl[ti][e];
          acc[e][0] = fmaf(g, x0, acc[e][0]);
          acc[e][1] = fmaf(g, x1, acc[e][1]);
          acc[e][2] = fmaf(g, x2, acc[e][2]);
          acc[e][3] = fmaf(g, x3, acc[e][3]);
        }
      }
    }
  }
  if (col < d) {
#pragma unroll
    for (int e = 0; e < kWgE; ++e) {
      if (e0 + e < E) {
        float4 v = make_float4(acc[e][0], acc[e][1], acc[e][2], acc[e][3]);
        *reinterpret_cast<float4*>(part + ((long)blockIdx.x * E + e0 + e) * d + col) = v;
      }
    }
  }
  if (blockIdx.y == 0 && threadIdx.x < kWgE && e0 + threadIdx.x < E)
    part_bias[(long)blockIdx.x * E + e0 + threadIdx.x] = bacc;
}

// 16 lanes per output element, each summing a strided subset of the block partials,
// then a 16-lane shuffle reduction (fixed order: deterministic).
__global__ void __launch_bounds__(256) router_wgrad_reduce(const float* __restrict__ part,
                                                           const float* __restrict__ part_bias,
                                                           int nblk, int d, int E,
                                                           float* __restrict__ dwg,
                                                           float* __restrict__ dbias) {
  const long n = (long)E * d;
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long i = gid >> 4;
  const int sub = threadIdx.x & 15;
  float s = 0.f, sb = 0.f;
  if (i < n)
    for (int b = sub; b < nblk; b += 16) s += part[(long)b * n + i];
  if (dbias && i < E)
    for (int b = sub; b < nblk; b += 16) sb += part_bias[(long)b * E + i];
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if (sub == 0 && i < n) {
    dwg[i] = s;
    if (dbias && i < E) dbias[i] = sb;
  }
}

__global__ void copy_segments_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, int d,
                                     const int32_t* __restrict__ src,
                                     const int32_t* __restrict__ dst,
                                     const int32_t* __restrict__ cnt) {
  const int g = blockIdx.y;
  const int nch = d / 8;
  const long n = cnt[g];
  const long s0 = src[g], d0 = dst[g];
  const long total = n * nch;
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long)gridDim.x * blockDim.x) {
    const long r = q / nch, c = q % nch;
    st_v4(out + (d0 + r) * nch + c, ld_nc_v4(in + (s0 + r) * nch + c));
  }
}

static int row_grid(long items) {
  const long want = (items + kRowWarps - 1) / kRowWarps;
  const long cap = (long)lzh::num_sms() * 16;  // 16 x 256-thread CTAs resident per SM max
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace lz

using namespace lz;

static long pad_items(int E, const int32_t* recv_m, const int32_t* recv_off, int align_hint) {
  (void)recv_m;
  (void)recv_off;
  return (long)E * align_hint;  // upper bound of pad rows handled per expert pass
}

// Pad rows are enumerated per expert inside zero_pad_rows; we launch enough warp
// items to cover the worst case of (align-1) pad rows per expert, align = 128.
static constexpr int kPadAlign = 256;  // >= the largest GEMM row alignment (lz_gemm_row_align)

static lz_status pack_impl(const void* x, int Tn, int d, int k, const int32_t* row,
                           const int32_t* prank, const unsigned long long* peers, void* out, int E,
                           const int32_t* recv_m, const int32_t* recv_off, void* stream) {
  if (Tn < 0 || d <= 0 || d % 8 || k < 1 || k > LZ_MAX_TOPK || E < 0) return LZ_ERR_ARG;
  if (Tn > 0 && (!x || !row || !out)) return LZ_ERR_ARG;
  if (E > 0 && (!recv_m || !recv_off || !out)) return LZ_ERR_ARG;
  const long npad = E > 0 ? pad_items(E, recv_m, recv_off, kPadAlign) : 0;
  if (Tn + npad == 0) return LZ_OK;
  pack_kernel<<<row_grid(Tn + npad), kRowThreads, 0, (cudaStream_t)stream>>>(
      (const uint4*)x, Tn, d, k, row, prank, peers, (uint4*)out, E, recv_m, recv_off, npad);
  return lzh::check_launch();
}

extern "C" lz_status lz_pack(const void* x, int Tn, int d, int k, const int32_t* row, void* out,
                             int E, const int32_t* recv_m, const int32_t* recv_off,
                             void* stream) {
  return pack_impl(x, Tn, d, k, row, nullptr, nullptr, out, E, recv_m, recv_off, stream);
}

extern "C" lz_status lz_pack_p2p(const void* x, int Tn, int d, int k, const int32_t* dest_rank,
                                 const int32_t* dest_row, const unsigned long long* peers,
                                 void* own, int E, const int32_t* recv_m,
                                 const int32_t* recv_off, void* stream) {
  if (!peers || !dest_rank) return LZ_ERR_ARG;
  return pack_impl(x, Tn, d, k, dest_row, dest_rank, peers, own, E, recv_m, recv_off, stream);
}

static lz_status combine_impl(const void* y, const int32_t* row, const int32_t* prank,
                              const unsigned long long* peers, const float* w, int Tn, int d,
                              int k, void* out, void* stream) {
  if (Tn < 0 || d <= 0 || d % 8 || k < 1 || k > LZ_MAX_TOPK) return LZ_ERR_ARG;
  if (Tn == 0) return LZ_OK;
  if ((!y && !peers) || !row || !w || !out) return LZ_ERR_ARG;
  combine_kernel<<<row_grid(Tn), kRowThreads, 0, (cudaStream_t)stream>>>(
      (const uint4*)y, row, prank, peers, w, Tn, d, k, (uint4*)out);
  return lzh::check_launch();
}

extern "C" lz_status lz_combine(const void* y, const int32_t* row, const float* w, int Tn, int d,
                                int k, void* out, void* stream) {
  return combine_impl(y, row, nullptr, nullptr, w, Tn, d, k, out, stream);
}

extern "C" lz_status lz_combine_p2p(const unsigned long long* peers_y, const int32_t* dest_rank,
                                    const int32_t* dest_row, const float* w, int Tn, int d,
                                    int k, void* out, void* stream) {
  if (!peers_y || !dest_rank) return LZ_ERR_ARG;
  return combine_impl(nullptr, dest_row, dest_rank, peers_y, w, Tn, d, k, out, stream);
}

static lz_status combine_bwd_impl(const void* dout, const void* y, const int32_t* row,
                                  const int32_t* prank, const unsigned long long* peers_y,
                                  const unsigned long long* peers_dy, const float* w, int Tn,
                                  int d, int k, void* dy, float* dw, int E,
                                  const int32_t* recv_m, const int32_t* recv_off, void* stream) {
  if (Tn < 0 || d <= 0 || d % 8 || k < 1 || k > LZ_MAX_TOPK || E < 0) return LZ_ERR_ARG;
  if (Tn > 0 && (!dout || (!y && !peers_y) || !row || !w || (!dy && !peers_dy) || !dw))
    return LZ_ERR_ARG;
  if (E > 0 && (!recv_m || !recv_off || !dy)) return LZ_ERR_ARG;
  const long npad = E > 0 ? pad_items(E, recv_m, recv_off, kPadAlign) : 0;
  if (Tn + npad == 0) return LZ_OK;
  combine_bwd_kernel<<<row_grid(Tn + npad), kRowThreads, 0, (cudaStream_t)stream>>>(
      (const uint4*)dout, (const uint4*)y, row, prank, peers_y, peers_dy, w, Tn, d, k, (uint4*)dy,
      dw, E, recv_m, recv_off, npad);
  return lzh::check_launch();
}

extern "C" lz_status lz_combine_bwd(const void* dout, const void* y, const int32_t* row,
                                    const float* w, int Tn, int d, int k, void* dy, float* dw,
                                    int E, const int32_t* recv_m, const int32_t* recv_off,
                                    void* stream) {
  return combine_bwd_impl(dout, y, row, nullptr, nullptr, nullptr, w, Tn, d, k, dy, dw, E, recv_m,
                          recv_off, stream);
}

extern "C" lz_status lz_combine_bwd_p2p(const void* dout, const unsigned long long* peers_y,
                                        const unsigned long long* peers_dy,
                                        const int32_t* dest_rank, const int32_t* dest_row,
                                        const float* w, int Tn, int d, int k, float* dw,
                                        void* own_dy, int E, const int32_t* recv_m,
                                        const int32_t* recv_off, void* stream) {
  if (!peers_y || !peers_dy || !dest_rank) return LZ_ERR_ARG;
  return combine_bwd_impl(dout, nullptr, dest_row, dest_rank, peers_y, peers_dy, w, Tn, d, k,
                          own_dy, dw, E, recv_m, recv_off, stream);
}

static lz_status dispatch_bwd_impl(const void* dxe, const int32_t* row, const int32_t* prank,
                                   const unsigned long long* peers, int Tn, int d, int k,
                                   const float* probs, const int32_t* idx, const float* dw,
                                   const void* wg, int E, int renorm, void* dx, float* dlogits,
                                   void* stream) {
  if (Tn < 0 || d <= 0 || d % 8 || k < 1 || k > LZ_MAX_TOPK || E < 1 || E > 64)
    return LZ_ERR_ARG;
  if (Tn == 0) return LZ_OK;
  if ((!dxe && !peers) || !row || !probs || !idx || !dw || !dx || !dlogits) return LZ_ERR_ARG;
  if (d % 64) return LZ_ERR_UNSUPPORTED;
  dispatch_bwd_kernel<<<row_grid((Tn + kDT - 1) / kDT), kRowThreads, 0, (cudaStream_t)stream>>>(
      (const uint4*)dxe, row, prank, peers, Tn, d, k, probs, idx, dw, (const __nv_bfloat16*)wg, E,
      renorm, (uint4*)dx, dlogits);
  return lzh::check_launch();
}

extern "C" lz_status lz_dispatch_bwd(const void* dxe, const int32_t* row, int Tn, int d, int k,
                                     const float* probs, const int32_t* idx, const float* dw,
                                     const void* wg, int E, int renorm, void* dx,
                                     float* dlogits, void* stream) {
  return dispatch_bwd_impl(dxe, row, nullptr, nullptr, Tn, d, k, probs, idx, dw, wg, E, renorm, dx,
                           dlogits, stream);
}

extern "C" lz_status lz_dispatch_bwd_p2p(const unsigned long long* peers_dxe,
                                         const int32_t* dest_rank, const int32_t* dest_row,
                                         int Tn, int d, int k, const float* probs,
                                         const int32_t* idx, const float* dw, const void* wg,
                                         int E, int renorm, void* dx, float* dlogits,
                                         void* stream) {
  if (!peers_dxe || !dest_rank) return LZ_ERR_ARG;
  return dispatch_bwd_impl(nullptr, dest_row, dest_rank, peers_dxe, Tn, d, k, probs, idx, dw, wg,
                           E, renorm, dx, dlogits, stream);
}

static int wgrad_nblk(int Tn) {
  int n = 2 * lzh::num_sms();
  long per = (Tn + n - 1) / n;
  if (per < 64) n = (Tn + 63) / 64;
  return n < 1 ? 1 : n;
}

extern "C" size_t lz_router_wgrad_ws_bytes(int Tn, int d, int E) {
  const size_t nblk = (size_t)wgrad_nblk(Tn);
  return nblk * (size_t)E * d * sizeof(float) + nblk * (size_t)E * sizeof(float) + 256;
}

extern "C" lz_status lz_router_wgrad(const float* dlogits, const void* x, int Tn, int d, int E,
                                     float* dwg, float* dbias, void* ws, size_t ws_bytes,
                                     void* stream) {
  if (Tn < 0 || d <= 0 || d % 4 || E < 1 || !dwg) return LZ_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (Tn == 0) {
    cudaMemsetAsync(dwg, 0, sizeof(float) * E * d, s);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * E, s);
    return lzh::check_launch();
  }
  if (!dlogits || !x || !ws) return LZ_ERR_ARG;
  if (ws_bytes < lz_router_wgrad_ws_bytes(Tn, d, E)) return LZ_ERR_WORKSPACE;
  const int nblk = wgrad_nblk(Tn);
  float* part = (float*)ws;
  float* part_bias = part + (size_t)nblk * E * d;
  dim3 grid(nblk, (d + 1023) / 1024, (E + kWgE - 1) / kWgE);
  router_wgrad_partial<<<grid, 256, 0, s>>>(dlogits, (const __nv_bfloat16*)x, Tn, d, E, part,
                                            part_bias);
  lz_status st = lzh::check_launch();
  if (st != LZ_OK) return st;
  const long n = (long)E * d;
  router_wgrad_reduce<<<(int)((16 * n + 255) / 256), 256, 0, s>>>(part, part_bias, nblk, d, E,
                                                                  dwg, dbias);
  return lzh::check_launch();
}

extern "C" lz_status lz_copy_segments(const void* in, void* out, int d, int nseg,
                                      const int32_t* src, const int32_t* dst, const int32_t* cnt,
                                      int max_cnt, void* stream) {
  if (d <= 0 || d % 8 || nseg < 0 || max_cnt < 0) return LZ_ERR_ARG;
  if (nseg == 0 || max_cnt == 0) return LZ_OK;
  if (!in || !out || !src || !dst || !cnt) return LZ_ERR_ARG;
  const long per = (long)max_cnt * (d / 8);
  int gx = (int)((per + 255) / 256);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, nseg);
  copy_segments_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint4*)in, (uint4*)out, d,
                                                               src, dst, cnt);
  return lzh::check_launch();
}

__global__ void invert_permutation_kernel(const int32_t* __restrict__ index, int n,
                                          int32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[__ldg(index + i)] = i;
}

extern "C" lz_status lz_invert_permutation(const int32_t* index, int n, int32_t* out,
                                           void* stream) {
  if (n < 0) return LZ_ERR_ARG;
  if (n == 0) return LZ_OK;
  if (!index || !out) return LZ_ERR_ARG;
  invert_permutation_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(index, n, out);
  return lzh::check_launch();
}
