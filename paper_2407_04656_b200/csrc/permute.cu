// permute.cu -- K3 pack, K7 combine, K8 backward permutes, router weight grad.
//
// All of these are HBM-bound row movers: one warp per token row, 16-byte
// vectorised coalesced loads/stores, 4 vectors in flight per lane, streaming
// (L1::no_allocate) loads for read-once activations.  Reference semantics:
//   pack     Alg. 1 reshuffle: token rows go to the send/receive
//            slot the planner assigned (dispatch.py:199-237 gives the index only)
//   combine  PAPER.md:99 weighted sum of the k expert outputs (fixed s order)
#include "common.cuh"

#ifndef LZ_D2_STAGES
#define LZ_D2_STAGES 2
#endif
#ifndef LZ_D2_BLOCKS
#define LZ_D2_BLOCKS 4
#endif

namespace lz {

constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / 32;
constexpr int kVec = 4;  // uint4 per lane in flight

__device__ __forceinline__ void zero_pad_rows(void* out, int d, int E, const int32_t* recv_m,
                                              const int32_t* recv_off, long item, long n_items,
                                              int lane, long long* ret_own = nullptr) {
  // item enumerates (expert, pad row) pairs; pad rows are [off[e]+m[e], off[e+1])
  (void)n_items;
  const int nch = d / 8;
  for (int e = 0; e < E; ++e) {
    const long start = (long)recv_off[e] + recv_m[e];
    const long cnt = (long)recv_off[e + 1] - start;
    if (item < cnt) {
      uint4* dst = reinterpret_cast<uint4*>(out) + (start + item) * nch;
      for (int c = lane; c < nch; c += 32) st_v4(dst + c, make_uint4(0, 0, 0, 0));
      if (ret_own && lane == 0) ret_own[start + item] = -1;   // pad row: no return target
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

// ret_peers (optional): every rank's return map; the owner row receiving assignment
// p = t*k + s of this rank records (my_rank << 32 | ret_row[p]) -- ret_row = the send
// slot, so each (owner, expert) segment maps to a contiguous row range here and the
// owner's GEMM epilogue can TMA-store the expert output straight back into this rank's
// return buffer.
__global__ void __launch_bounds__(kRowThreads) pack_kernel(
    const uint4* __restrict__ x, int Tn, int d, int k, const int32_t* __restrict__ row,
    const int32_t* __restrict__ prank, const unsigned long long* __restrict__ peers,
    uint4* __restrict__ out, int E, const int32_t* __restrict__ recv_m,
    const int32_t* __restrict__ recv_off, long n_pad_items,
    const unsigned long long* __restrict__ ret_peers, long long* __restrict__ ret_own,
    int my_rank, const int32_t* __restrict__ ret_row) {
  const int lane = threadIdx.x % 32;
  pdl_prologue();
  const long gw = (long)blockIdx.x * kRowWarps + threadIdx.x / 32;
  const long nw = (long)gridDim.x * kRowWarps;
  const int nch = d / 8;
  for (long t = gw; t < Tn + n_pad_items; t += nw) {
    if (t >= Tn) {
      zero_pad_rows(out, d, E, recv_m, recv_off, t - Tn, n_pad_items, lane, ret_own);
      continue;
    }
    const int my_row = lane < k ? __ldg(row + t * k + lane) : 0;
    const int my_rk = (peers && lane < k) ? __ldg(prank + t * k + lane) : 0;
    if (ret_peers && lane < k)
      reinterpret_cast<long long*>(ret_peers[my_rk])[my_row] =
          ((long long)my_rank << 32) | (long long)__ldg(ret_row + t * k + lane);
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

// Bulk-copy (TMA engine) variant of the pack: rows go HBM -> smem -> HBM through
// cp.async.bulk, the SM only issues the copies.  Lane 0 of each warp drives a ring of
// kPbSlots row slots: the loads of the next kPbSlots - 1 tokens of the warp are in flight
// while the current token's row is stored to its k destinations (peers' buffers over
// NVLink included) by bulk stores; a slot is refilled once its stores have read it
// (bulk_group accounting).  Lanes < k write the return-map entries; pad rows are zeroed
// with plain stores as in pack_kernel.  Selected with LZ_PACK_BULK=1 (A/B: DESIGN.md 4).
constexpr int kPbWarps = 8, kPbSlots = 8;
__device__ __forceinline__ uint32_t pb_smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__global__ void __launch_bounds__(32 * kPbWarps, 1) pack_bulk_kernel(
    const uint4* __restrict__ x, int Tn, int d, int k, const int32_t* __restrict__ row,
    const int32_t* __restrict__ prank, const unsigned long long* __restrict__ peers,
    uint4* __restrict__ out, int E, const int32_t* __restrict__ recv_m,
    const int32_t* __restrict__ recv_off, long n_pad_items,
    const unsigned long long* __restrict__ ret_peers, long long* __restrict__ ret_own,
    int my_rank, const int32_t* __restrict__ ret_row) {
  extern __shared__ __align__(128) uint8_t pb_smem[];
  __shared__ __align__(8) uint64_t pb_bar[kPbWarps][kPbSlots];
  pdl_prologue();
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const uint32_t rb = (uint32_t)d * 2;
  uint8_t* ring = pb_smem + (size_t)warp * kPbSlots * rb;
  const long gw = (long)blockIdx.x * kPbWarps + warp;
  const long nw = (long)gridDim.x * kPbWarps;
  const int nch = d / 8;
  if (lane == 0) {
    for (int j = 0; j < kPbSlots; ++j)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(pb_smem_u32(&pb_bar[warp][j])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto load = [&](long i) {   // token gw + i * nw into slot i % kPbSlots (lane 0)
    const long t = gw + i * nw;
    const int j = (int)(i % kPbSlots);
    const uint32_t bar = pb_smem_u32(&pb_bar[warp][j]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rb)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            pb_smem_u32(ring + (size_t)j * rb)),
        "l"(x + t * nch), "r"(rb), "r"(bar)
        : "memory");
  };
  const long ntok = gw < Tn ? (Tn - gw + nw - 1) / nw : 0;   // this warp's tokens
  if (lane == 0)
    for (long i = 0; i < kPbSlots && i < ntok; ++i) load(i);
  uint32_t phases = 0;   // one parity bit per slot
  for (long i = 0; i < ntok; ++i) {
    const long t = gw + i * nw;
    const int my_row = lane < k ? __ldg(row + t * k + lane) : 0;
    const int my_rk = (peers && lane < k) ? __ldg(prank + t * k + lane) : 0;
    if (ret_peers && lane < k)
      reinterpret_cast<long long*>(ret_peers[my_rk])[my_row] =
          ((long long)my_rank << 32) | (long long)__ldg(ret_row + t * k + lane);
    long dst[LZ_MAX_TOPK];
    for (int s2 = 0; s2 < k; ++s2) {
      const long r = __shfl_sync(0xffffffffu, my_row, s2);
      const int rk = __shfl_sync(0xffffffffu, my_rk, s2);
      dst[s2] = (long)((peers ? reinterpret_cast<uint4*>(peers[rk]) : out) + r * nch);
    }
    if (lane == 0) {
      const int j = (int)(i % kPbSlots);
      const uint32_t bar = pb_smem_u32(&pb_bar[warp][j]);
      const uint32_t par = (phases >> j) & 1u;
      uint32_t done = 0;
      do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(par)
            : "memory");
      } while (!done);
      phases ^= 1u << j;
      const uint32_t src = pb_smem_u32(ring + (size_t)j * rb);
      for (int s2 = 0; s2 < k; ++s2)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst[s2]),
                     "r"(src), "r"(rb)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // refill the previous token's slot: its stores (the second most recent group) have
      // finished reading it once at most one group is still reading
      if (i >= 1 && i - 1 + kPbSlots < ntok) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        load(i - 1 + kPbSlots);
      }
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
  // pad rows of the expert-major layout (and their return-map entries)
  for (long q = gw; q < n_pad_items; q += nw)
    zero_pad_rows(out, d, E, recv_m, recv_off, q, n_pad_items, lane, ret_own);
}

__global__ void __launch_bounds__(kRowThreads) combine_kernel(
    const uint4* __restrict__ y, const int32_t* __restrict__ row, const int32_t* __restrict__ prank,
    const unsigned long long* __restrict__ peers, const float* __restrict__ w, int Tn, int d, int k,
    uint4* __restrict__ out) {
  const int lane = threadIdx.x % 32;
  pdl_prologue();
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

#ifndef LZ_CBWD_MINB
#define LZ_CBWD_MINB 2
#endif
#ifndef LZ_CBWD_VEC
#define LZ_CBWD_VEC 4
#endif
__global__ void __launch_bounds__(kRowThreads, LZ_CBWD_MINB) combine_bwd_kernel(
    const uint4* __restrict__ dout, const uint4* __restrict__ y, const int32_t* __restrict__ row,
    const int32_t* __restrict__ prank, const unsigned long long* __restrict__ peers_y,
    const unsigned long long* __restrict__ peers_dy,
    const float* __restrict__ w, int Tn, int d, int k, uint4* __restrict__ dy,
    float* __restrict__ dw, int E, const int32_t* __restrict__ recv_m,
    const int32_t* __restrict__ recv_off, long n_pad_items,
    const int32_t* __restrict__ yrow) {
  pdl_prologue();
  // yrow (optional): y is this rank's own return buffer and assignment p's expert output
  // sits at row yrow[p] (written by the owners' scattering GEMM epilogue); dy still goes
  // to the owner's row
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
    const int my_yrow = (yrow && lane < k) ? __ldg(yrow + t * k + lane) : 0;
    const float my_w = lane < k ? __ldg(w + t * k + lane) : 0.f;
    const int my_rk = ((peers_y || peers_dy) && lane < k) ? __ldg(prank + t * k + lane) : 0;
    float dot[LZ_MAX_TOPK];
#pragma unroll
    for (int s = 0; s < LZ_MAX_TOPK; ++s) dot[s] = 0.f;
    for (int c0 = lane; c0 < nch; c0 += 32 * kVec) {
      if (k == 2) {
        // common top-2: the dout chunk and BOTH expert rows in flight before any math
        constexpr int kV2 = LZ_CBWD_VEC;
        uint4 gv[kV2], yv[2][kV2];
        const uint4* ys[2];
        uint4* dys[2];
        float ws[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const long r = __shfl_sync(0xffffffffu, my_row, s);
          ws[s] = __shfl_sync(0xffffffffu, my_w, s);
          ys[s] = yrow ? y + (long)__shfl_sync(0xffffffffu, my_yrow, s) * nch
                       : row_base(const_cast<uint4*>(y), peers_y, my_rk, s) + r * nch;
          dys[s] = row_base(dy, peers_dy, my_rk, s) + r * nch;
        }
        for (int cb = c0; cb < c0 + 32 * kVec; cb += 32 * kV2) {
#pragma unroll
          for (int u = 0; u < kV2; ++u) {
            if (cb + 32 * u < nch) {
              gv[u] = ld_nc_v4(dout + t * nch + cb + 32 * u);
              yv[0][u] = ld_nc_v4(ys[0] + cb + 32 * u);
              yv[1][u] = ld_nc_v4(ys[1] + cb + 32 * u);
            }
          }
#pragma unroll
          for (int u = 0; u < kV2; ++u) {
            if (cb + 32 * u < nch) {
              float gf[8];
              bf16x8_to_f32(gv[u], gf);
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                float f[8], o[8];
                bf16x8_to_f32(yv[s][u], f);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                  dot[s] = fmaf(gf[q], f[q], dot[s]);
                  o[q] = ws[s] * gf[q];
                }
                st_v4(dys[s] + cb + 32 * u, f32_to_bf16x8(o));
              }
            }
          }
        }
        continue;
      }
      float g[kVec][8];
#pragma unroll
      for (int u = 0; u < kVec; ++u)
        if (c0 + 32 * u < nch) bf16x8_to_f32(ld_nc_v4(dout + t * nch + c0 + 32 * u), g[u]);
#pragma unroll
      for (int s = 0; s < LZ_MAX_TOPK; ++s) {
        if (s >= k) break;
        const long r = __shfl_sync(0xffffffffu, my_row, s);
        const float ws = __shfl_sync(0xffffffffu, my_w, s);
        const uint4* ys = yrow ? y + (long)__shfl_sync(0xffffffffu, my_yrow, s) * nch
                               : row_base(const_cast<uint4*>(y), peers_y, my_rk, s) + r * nch;
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

// Gate backward (softmax + top-k (+renorm)) and dispatch backward, fused per 16-token
// tile: dlogits from probs / idx / dw, then dx = sum_s dxe[row(t, s)] + dlogits . wg with
// the router term on the tensor cores (mma.sync m16n8k16, dlogits split into bf16 hi + lo
// so the product keeps ~16 mantissa bits).
constexpr int kDT = 16;
__device__ __forceinline__ uint32_t bf16pair(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(pred ? 16 : 0)
               : "memory");
}
// Register-direct variant.  The router-term MMA's output columns are permuted so that
// each lane's C fragment covers 8 CONTIGUOUS row columns: in the 32-column block b, lane
// (g, t4) of n8 tile nt holds columns b*32 + t4*8 + 2*nt + {0, 1} for tokens g and g + 8
// (the B fragment of n8 tile nt therefore loads the router-weight columns
// b*32 + (n >> 1)*8 + 2*nt + (n & 1), n = 0..7).  The lane then adds its tokens' gathered
// expert rows (one 16-byte load per (token, s, block)) and stores dx -- no shared-memory
// round trip of the router term, no column-pass barriers.  Phase A (dlogits) runs on all
// 32 lanes: lane pair (2 ti, 2 ti + 1) owns token ti, each lane half of its experts.
constexpr int kD2Warps = 4;
constexpr int kD2Stages = LZ_D2_STAGES;
constexpr int kD2Smem = kD2Warps * kD2Stages * 8 * 32 * 16;
__device__ __forceinline__ uint4 ld_shared_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
// Phase-A inputs of one task (lane pair 2 ti, 2 ti + 1 = token ti; lane half h holds the
// probabilities of experts [h EH, (h + 1) EH)); loaded one task ahead
template <int EH>
struct DbwdIn {
  int id[2], row[2], rk[2];
  float dw[2], pr[EH];
};
template <int EH>
__device__ __forceinline__ void dbwd_load(DbwdIn<EH>& in, long t, int Tn, int k, int E, int h,
                                          const int32_t* __restrict__ idx,
                                          const float* __restrict__ dwv,
                                          const int32_t* __restrict__ row,
                                          const int32_t* __restrict__ prank,
                                          const float* __restrict__ probs, bool peers) {
  const bool ok = t < Tn;
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2) {
    const bool o = ok && s2 < k;
    in.id[s2] = o ? __ldg(idx + t * k + s2) : -1;
    in.dw[s2] = o ? __ldg(dwv + t * k + s2) : 0.f;
    in.row[s2] = o ? __ldg(row + t * k + s2) : 0;
    in.rk[s2] = (o && peers) ? __ldg(prank + t * k + s2) : 0;
  }
#pragma unroll
  for (int j = 0; j < EH; ++j) {
    const int e = h * EH + j;
    in.pr[j] = (ok && e < E) ? __ldg(probs + t * E + e) : 0.f;
  }
}
template <int KS, int ET>
__global__ void __launch_bounds__(32 * kD2Warps) dispatch_bwd_reg(
    const uint4* __restrict__ dxe, const int32_t* __restrict__ row,
    const int32_t* __restrict__ prank, const unsigned long long* __restrict__ peers, int Tn, int d,
    int k, const float* __restrict__ probs, const int32_t* __restrict__ idx,
    const float* __restrict__ dwv, const __nv_bfloat16* __restrict__ wg, int E_rt, int renorm,
    uint4* __restrict__ dx, float* __restrict__ dlogits, int nh) {
  const int E = ET > 0 ? ET : E_rt;
  constexpr int EP = KS * 16;                 // experts padded to the MMA k steps
  constexpr int EH = EP / 2;                  // experts per phase-A lane
  __shared__ __align__(16) float s_dl[kD2Warps][kDT][EP + 4];
  __shared__ long long s_src[kD2Warps][kDT][LZ_MAX_TOPK];
  extern __shared__ __align__(16) uint4 d2_ring[];   // [warps][stages][8 slots][32 lanes]
  pdl_prologue();
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const long gw = (long)blockIdx.x * kD2Warps + warp;
  const long nw = (long)gridDim.x * kD2Warps;
  const int nch = d / 8;
  const int g = lane >> 2, t4 = lane & 3;
  const int ti = lane >> 1, h = lane & 1;     // phase-A token / expert half
  const uint32_t* wT = reinterpret_cast<const uint32_t*>(wg);
  const long ntask = (long)((Tn + kDT - 1) / kDT) * nh;
  const int dcols = d / nh;                   // columns of one task
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(d2_ring) +
                        (uint32_t)(warp * kD2Stages * 8 * 32 * 16) + lane * 16;
  DbwdIn<EH> nxt;
  if (gw < ntask)
    dbwd_load<EH>(nxt, (gw / nh) * kDT + ti, Tn, k, E, h, idx, dwv, row, prank, probs,
                  peers != nullptr);
  for (long task = gw; task < ntask; task += nw) {
    const long t0 = (task / nh) * kDT;
    const int half = (int)(task % nh);
    const DbwdIn<EH> in = nxt;
    if (task + nw < ntask)   // next task's phase-A inputs in flight during this task
      dbwd_load<EH>(nxt, ((task + nw) / nh) * kDT + ti, Tn, k, E, h, idx, dwv, row, prank,
                    probs, peers != nullptr);
    // ---- phase A: dlogits (dp_e is non-zero only at the k routed experts:
    //   dot = sum_s g_s p_{idx_s},  dl_e = p_e (dp_e - dot), g_s = dw_s or its renorm form)
    {
      const long t = t0 + ti;
      float dl[EH];
      // p_{idx_s} from the lane of the pair that holds expert idx_s (all lanes shuffle)
      float pin[2];
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        float mine = 0.f;
#pragma unroll
        for (int j = 0; j < EH; ++j)
          if (in.id[s2] == h * EH + j) mine = in.pr[j];
        const float other = __shfl_xor_sync(0xffffffffu, mine, 1);
        pin[s2] = (in.id[s2] >= 0 && in.id[s2] / EH == h) ? mine : other;
      }
      if (t < Tn) {
        int ids[LZ_MAX_TOPK];
        float gs[LZ_MAX_TOPK], ps[LZ_MAX_TOPK];
#pragma unroll
        for (int s2 = 0; s2 < LZ_MAX_TOPK; ++s2) {
          ids[s2] = -1;
          gs[s2] = ps[s2] = 0.f;
          if (s2 >= k) continue;
          int e, rr, rk;
          float p;
          if (s2 < 2) {
            e = in.id[s2];
            gs[s2] = in.dw[s2];
            rr = in.row[s2];
            rk = in.rk[s2];
            p = pin[s2];
          } else {
            e = __ldg(idx + t * k + s2);
            gs[s2] = __ldg(dwv + t * k + s2);
            rr = __ldg(row + t * k + s2);
            rk = peers ? __ldg(prank + t * k + s2) : 0;
            p = __ldg(probs + t * E + e);
          }
          ids[s2] = e;
          ps[s2] = p;
          if (h == 0) {
            const uint4* base = peers ? reinterpret_cast<const uint4*>(peers[rk]) : dxe;
            s_src[warp][ti][s2] = (long long)(base + (long)rr * nch);
          }
        }
        const float dot = gate_bwd_coefs(k, renorm, ps, gs);
#pragma unroll
        for (int j = 0; j < EH; ++j) dl[j] = gate_bwd_dl(in.pr[j], h * EH + j, dot, ids, gs);
        if (half == 0) {
          if (ET > 0 && ET % 8 == 0 && EH % 4 == 0) {
#pragma unroll
            for (int j = 0; j < EH; j += 4)
              if (h * EH + j < E)
                *reinterpret_cast<float4*>(dlogits + t * E + h * EH + j) =
                    make_float4(dl[j], dl[j + 1], dl[j + 2], dl[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < EH; ++j)
              if (h * EH + j < E) dlogits[t * E + h * EH + j] = dl[j];
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < EH; ++j) dl[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < EH; j += 4)
        *reinterpret_cast<float4*>(&s_dl[warp][ti][h * EH + j]) =
            make_float4(dl[j], dl[j + 1], dl[j + 2], dl[j + 3]);
    }
    __syncwarp();
    const int nt = (int)min((long)kDT, Tn - t0);
    const bool v0 = g < nt, v1 = g + 8 < nt;
    // A fragments: dlogits rows (tokens) x experts, bf16 hi + lo
    uint32_t ah[KS][4], al[KS][4];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int e0 = ks * 16 + 2 * t4;
      const float v[8] = {s_dl[warp][g][e0],         s_dl[warp][g][e0 + 1],
                          s_dl[warp][g + 8][e0],     s_dl[warp][g + 8][e0 + 1],
                          s_dl[warp][g][e0 + 8],     s_dl[warp][g][e0 + 9],
                          s_dl[warp][g + 8][e0 + 8], s_dl[warp][g + 8][e0 + 9]};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float x0 = v[2 * r], x1 = v[2 * r + 1];
        ah[ks][r] = bf16pair(x0, x1);
        const float h0 = __uint_as_float(ah[ks][r] << 16);
        const float h1 = __uint_as_float(ah[ks][r] & 0xffff0000u);
        al[ks][r] = bf16pair(x0 - h0, x1 - h1);
      }
    }
    const uint4* src0[2];
    const uint4* src1[2];
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      src0[s2] = (v0 && s2 < k) ? reinterpret_cast<const uint4*>(s_src[warp][g][s2]) : nullptr;
      src1[s2] = (v1 && s2 < k) ? reinterpret_cast<const uint4*>(s_src[warp][g + 8][s2])
                                : nullptr;
    }
    // ---- phase B: 64 columns (two 32-column blocks) per pass.  The gathered rows of the
    // next kD2Stages - 1 passes are in flight as cp.async copies into this lane's own ring
    // slots (slot j = token half * 4 + block * 2 + s; lane-private, so no warp barrier) ----
    const int cbeg = half * dcols;
    const int npass = dcols / 64;
    auto issue = [&](int pass) {
      const uint32_t st = ring + (uint32_t)((pass % kD2Stages) * 8 * 32 * 16);
      const int c0 = (cbeg >> 3) + pass * 8 + t4;
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          cp_async16(st + (uint32_t)((b * 2 + s2) * 512),
                     src0[s2] ? (const void*)(src0[s2] + c0 + 4 * b) : (const void*)dx,
                     src0[s2] != nullptr);
          cp_async16(st + (uint32_t)((4 + b * 2 + s2) * 512),
                     src1[s2] ? (const void*)(src1[s2] + c0 + 4 * b) : (const void*)dx,
                     src1[s2] != nullptr);
        }
    };
#pragma unroll
    for (int i = 0; i < kD2Stages - 1; ++i) {
      if (i < npass) issue(i);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int pass = 0; pass < npass; ++pass) {
      if (pass + kD2Stages - 1 < npass) issue(pass + kD2Stages - 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      const int cb = cbeg + pass * 64;
      const int c0 = (cb >> 3) + t4;        // chunk of block 0; block 1 is c0 + 4
      float acc[2][4][4];
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[b][n][q] = 0.f;
      if (wg) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int e0 = ks * 16 + 2 * t4;
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int n = 0; n < 4; ++n) {
              const long col = cb + b * 32 + (g >> 1) * 8 + 2 * n + (g & 1);
              const uint32_t w0 = e0 < E ? __ldg(wT + ((col * E + e0) >> 1)) : 0u;
              const uint32_t w1 = e0 + 8 < E ? __ldg(wT + ((col * E + e0 + 8) >> 1)) : 0u;
              mma16816(acc[b][n], ah[ks][0], ah[ks][1], ah[ks][2], ah[ks][3], w0, w1);
              mma16816(acc[b][n], al[ks][0], al[ks][1], al[ks][2], al[ks][3], w0, w1);
            }
        }
      }
      asm volatile("cp.async.wait_group %0;" ::"n"(kD2Stages - 1) : "memory");
      const uint32_t st = ring + (uint32_t)((pass % kD2Stages) * 8 * 32 * 16);
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        float f0[8], f1[8];
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          f0[2 * n] = acc[b][n][0];
          f0[2 * n + 1] = acc[b][n][1];
          f1[2 * n] = acc[b][n][2];
          f1[2 * n + 1] = acc[b][n][3];
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          float a[8], c[8];
          bf16x8_to_f32(ld_shared_u4(st + (uint32_t)((b * 2 + s2) * 512)), a);
          bf16x8_to_f32(ld_shared_u4(st + (uint32_t)((4 + b * 2 + s2) * 512)), c);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            f0[q] += a[q];
            f1[q] += c[q];
          }
        }
        if (k > 2) {
          for (int s2 = 2; s2 < k; ++s2) {
            float a[8];
            if (v0) {
              bf16x8_to_f32(ld_nc_v4(reinterpret_cast<const uint4*>(s_src[warp][g][s2]) +
                                     c0 + 4 * b),
                            a);
#pragma unroll
              for (int q = 0; q < 8; ++q) f0[q] += a[q];
            }
            if (v1) {
              bf16x8_to_f32(ld_nc_v4(reinterpret_cast<const uint4*>(s_src[warp][g + 8][s2]) +
                                     c0 + 4 * b),
                            a);
#pragma unroll
              for (int q = 0; q < 8; ++q) f1[q] += a[q];
            }
          }
        }
        if (v0) st_v4(dx + (t0 + g) * nch + c0 + 4 * b, f32_to_bf16x8(f0));
        if (v1) st_v4(dx + (t0 + g + 8) * nch + c0 + 4 * b, f32_to_bf16x8(f1));
      }
    }
    __syncwarp();   // s_dl / s_src of this task consumed before the next task's phase A
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

// Column-sliced tensor-core variant (the default for d % 128 == 0): block (r, c, z) reduces
// token range r for the 128 columns [128 c, +128) and experts [16 z, +16); warp w owns 32
// of the columns (two m16 tiles), so the accumulators are 32 registers.  The token ranges
// are few (blocks per SM * SMs / slices), so the partials are E * d * 4 bytes per range
// (cfg2: 3.6 MB).  Per step the block stages kR2Tok x 128 bf16 of x and the kR2Tok x 16
// dlogits through a cp.async ring (precomputed strided addresses); the dlogits' hi / lo
// bf16 B fragments are built once per step by the whole block into shared memory, and the
// bias partial is summed by all threads.
// 64-token steps, 3 stages, 3 blocks per SM: measured best of (32|64|96|128 tokens) x
// (2..4 stages) x (1..6 blocks/SM) -- 30.0 us vs 32.1 us for 32-token steps at 6 blocks/SM
#ifndef LZ_R2_TOK
#define LZ_R2_TOK 64
#define LZ_R2_ST 3
#define LZ_R2_BLK 3
#endif
constexpr int kR2Cols = 128, kR2Row = kR2Cols + 8, kR2Stages = LZ_R2_ST, kR2Tok = LZ_R2_TOK;
constexpr int kR2StageBytes = kR2Tok * kR2Row * 2 + kR2Tok * 16 * 4;   // x tile + dlogits
constexpr int kR2Smem = kR2Stages * kR2StageBytes + (kR2Tok / 16) * 2 * 2 * 2 * 32 * 4;
__global__ void __launch_bounds__(128, LZ_R2_BLK) router_wgrad_tc2(const float* __restrict__ dlog,
                                                         const __nv_bfloat16* __restrict__ x,
                                                         int Tn, int d, int E,
                                                         float* __restrict__ part,
                                                         float* __restrict__ part_bias) {
  extern __shared__ __align__(16) uint8_t r2_smem[];
  pdl_prologue();
  constexpr int KG = kR2Tok / 16;   // 16-token k groups per step
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int g = lane >> 2, t4 = lane & 3;
  const int nrange = gridDim.x;
  const int cbase = blockIdx.y * kR2Cols;
  const int e0 = blockIdx.z * 16;
  const long per = ((long)(Tn + nrange - 1) / nrange + kR2Tok - 1) / kR2Tok * kR2Tok;
  const long t_begin = (long)blockIdx.x * per;
  const long t_end = min((long)Tn, t_begin + per);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(r2_smem);
  // B fragments of the step: [kg][n][h][hi / lo][32 lanes]
  uint32_t* s_bf = reinterpret_cast<uint32_t*>(r2_smem + kR2Stages * kR2StageBytes);
  // staging: kR2Tok rows x 256 B of x (16 pieces of 16 B per row) + kR2Tok x 16 dlogits.
  // Thread tid copies piece (tid & 15) of rows (tid >> 4) + 8 j: its global / shared
  // addresses advance by fixed strides, precomputed once
  const int ti0 = threadIdx.x >> 4, cc0 = threadIdx.x & 15;
  const __nv_bfloat16* xg0 = x + (t_begin + ti0) * d + cbase + cc0 * 8;
  const uint32_t sx_off = (uint32_t)((ti0 * kR2Row + cc0 * 8) * 2);
  // dlogits: one 16-byte piece (4 experts) per thread when a token's 16-expert slice is
  // 16-byte aligned (E % 4 == 0), else 4-byte copies
  const bool dl16 = (E % 4) == 0;
  const int dti = threadIdx.x >> 2, dq = threadIdx.x & 3;   // 32 tokens x 4 pieces
  auto stage = [&](int buf, long tt) {
    const uint32_t sx = sbase + (uint32_t)(buf * kR2StageBytes);
    const long rel = tt - t_begin;
    const __nv_bfloat16* xg = xg0 + rel * d;
#pragma unroll
    for (int j = 0; j < kR2Tok / 8; ++j) {
      const bool ok = tt + ti0 + 8 * j < t_end;
      cp_async16(sx + sx_off + (uint32_t)(8 * j * kR2Row * 2), ok ? (const void*)(xg + 8L * j * d)
                                                                 : (const void*)x,
                 ok);
    }
    const uint32_t sdl = sx + (uint32_t)(kR2Tok * kR2Row * 2);
    if (dl16) {
#pragma unroll
      for (int jj = 0; jj < kR2Tok / 32; ++jj) {
        const long t = tt + dti + 32 * jj;
        const bool ok = t < t_end && e0 + 4 * dq < E;
        cp_async16(sdl + (uint32_t)(((dti + 32 * jj) * 16 + 4 * dq) * 4),
                   ok ? (const void*)(dlog + t * E + e0 + 4 * dq) : (const void*)dlog, ok);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kR2Tok * 16 / 128; ++j) {
        const int q = threadIdx.x + j * 128;
        const int ti = q >> 4, ei = q & 15;
        const long t = tt + ti;
        const bool ok = t < t_end && e0 + ei < E;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sdl + (uint32_t)(q * 4)),
                     "l"(dlog + (ok ? t * E + e0 + ei : 0)), "r"(ok ? 4 : 0)
                     : "memory");
      }
    }
  };
  float acc[2][2][4];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[m][n][q] = 0.f;
  float bacc = 0.f;
  const long nsteps = t_end > t_begin ? (t_end - t_begin + kR2Tok - 1) / kR2Tok : 0;
#pragma unroll
  for (int i = 0; i < kR2Stages - 1; ++i) {
    if (i < nsteps) stage(i, t_begin + (long)i * kR2Tok);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // B-fragment builder roles of this thread: (n, h) = threadIdx.x / 32 for every k group
  const int bn = threadIdx.x >> 6, bh = (threadIdx.x >> 5) & 1;
  const int mi = lane >> 3, r = lane & 7;
  for (long i = 0; i < nsteps; ++i) {
    const int buf = (int)(i % kR2Stages);
    asm volatile("cp.async.wait_group %0;" ::"n"(kR2Stages - 2) : "memory");
    __syncthreads();   // step i landed for every thread; buffer (i - 1) % S free again
    {
      const long j = i + kR2Stages - 1;
      if (j < nsteps) stage((int)(j % kR2Stages), t_begin + j * kR2Tok);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const float* dl = reinterpret_cast<const float*>(r2_smem + buf * kR2StageBytes +
                                                     kR2Tok * kR2Row * 2);
#pragma unroll
    for (int kg = 0; kg < KG; ++kg) {
      // B fragment (experts n*8 + g; tokens k0, k0 + 1 with k0 = 16 kg + 2 t4 + 8 h), hi + lo
      const int k0 = 16 * kg + 2 * t4 + 8 * bh;
      const float v0 = dl[k0 * 16 + bn * 8 + g], v1 = dl[(k0 + 1) * 16 + bn * 8 + g];
      const uint32_t hi = bf16pair(v0, v1);
      const float h0 = __uint_as_float(hi << 16), h1 = __uint_as_float(hi & 0xffff0000u);
      s_bf[(((kg * 2 + bn) * 2 + bh) * 2 + 0) * 32 + lane] = hi;
      s_bf[(((kg * 2 + bn) * 2 + bh) * 2 + 1) * 32 + lane] = bf16pair(v0 - h0, v1 - h1);
    }
    if (blockIdx.y == 0) {
      // bias partial: thread (expert e = tid & 15, token group j = tid >> 4) adds its 4 of
      // the step's 32 tokens (all 128 threads, no serial 32-token loop in one warp)
      const int e = threadIdx.x & 15, j = threadIdx.x >> 4;
#pragma unroll
      for (int q = 0; q < kR2Tok / 8; ++q) bacc += dl[(j * (kR2Tok / 8) + q) * 16 + e];
    }
    __syncthreads();   // B fragments of step i visible
#pragma unroll
    for (int kg = 0; kg < KG; ++kg) {
      uint32_t bf[2][2][2];   // [n][h][hi / lo]
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int hl = 0; hl < 2; ++hl)
            bf[n][h][hl] = s_bf[(((kg * 2 + n) * 2 + h) * 2 + hl) * 32 + lane];
      // A fragments: ldmatrix.x4.trans of the 16 tokens x 16 columns submatrix
      const uint32_t abase =
          sbase + (uint32_t)(buf * kR2StageBytes) +
          (uint32_t)(((16 * kg + (mi >> 1) * 8 + r) * kR2Row + warp * 32 + (mi & 1) * 8) * 2);
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        uint32_t a0, a1, a2, a3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                     : "r"(abase + m * 32));
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          mma16816(acc[m][n], a0, a1, a2, a3, bf[n][0][0], bf[n][1][0]);
          mma16816(acc[m][n], a0, a1, a2, a3, bf[n][0][1], bf[n][1][1]);
        }
      }
    }
  }
  // partial[range][e][col]: C fragment rows = columns (g, g + 8), cols = experts (2t4, +1)
  float* pb = part + (long)blockIdx.x * E * d;
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int c = cbase + warp * 32 + m * 16 + g;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      const int e = e0 + n * 8 + 2 * t4;
      if (e < E) {
        pb[(long)e * d + c] = acc[m][n][0];
        pb[(long)e * d + c + 8] = acc[m][n][2];
      }
      if (e + 1 < E) {
        pb[(long)(e + 1) * d + c] = acc[m][n][1];
        pb[(long)(e + 1) * d + c + 8] = acc[m][n][3];
      }
    }
  }
  if (blockIdx.y == 0) {
    // the 8 token-group partials of each expert, summed in a fixed order
    __shared__ float s_b[8][16];
    s_b[threadIdx.x >> 4][threadIdx.x & 15] = bacc;
    __syncthreads();
    if (threadIdx.x < 16 && e0 + threadIdx.x < E) {
      float v = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) v += s_b[j][threadIdx.x];
      part_bias[(long)blockIdx.x * E + e0 + threadIdx.x] = v;
    }
  }
}

// Block = 8 warps x 32 consecutive output elements (coalesced 128-byte loads); warp w
// sums partials w, w + 8, ... and the 8 warp sums are added in a fixed order through
// shared memory (deterministic).  The trailing ceil(E/32) blocks reduce the bias partials.
__global__ void __launch_bounds__(256) router_wgrad_reduce(const float* __restrict__ part,
                                                           const float* __restrict__ part_bias,
                                                           int nblk, int d, int E,
                                                           float* __restrict__ dwg,
                                                           float* __restrict__ dbias) {
  __shared__ float s_sum[8][33];
  pdl_prologue();
  const long n = (long)E * d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long nmain = (n + 31) / 32;
  const bool bias_blk = blockIdx.x >= nmain;
  const long i = (bias_blk ? blockIdx.x - nmain : blockIdx.x) * 32 + lane;
  const long stride = bias_blk ? E : n;
  const float* src = bias_blk ? part_bias : part;
  const bool ok = bias_blk ? (dbias != nullptr && i < E) : i < n;
  float s = 0.f;
  if (ok) {
    int b = warp;
    for (; b + 24 < nblk; b += 32) {   // 4 independent loads in flight per iteration
      const float v0 = __ldg(src + (long)b * stride + i);
      const float v1 = __ldg(src + (long)(b + 8) * stride + i);
      const float v2 = __ldg(src + (long)(b + 16) * stride + i);
      const float v3 = __ldg(src + (long)(b + 24) * stride + i);
      s += v0;
      s += v1;
      s += v2;
      s += v3;
    }
    for (; b < nblk; b += 8) s += __ldg(src + (long)b * stride + i);
  }
  s_sum[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && ok) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_sum[w][lane];
    if (bias_blk) dbias[i] = t;
    else dwg[i] = t;
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
                           const int32_t* recv_m, const int32_t* recv_off, void* stream,
                           const unsigned long long* ret_peers = nullptr,
                           long long* ret_own = nullptr, int my_rank = 0,
                           const int32_t* ret_row = nullptr) {
  if (Tn < 0 || d <= 0 || d % 8 || k < 1 || k > LZ_MAX_TOPK || E < 0) return LZ_ERR_ARG;
  if (Tn > 0 && (!x || !row || !out)) return LZ_ERR_ARG;
  if (E > 0 && (!recv_m || !recv_off || !out)) return LZ_ERR_ARG;
  const long npad = E > 0 ? pad_items(E, recv_m, recv_off, kPadAlign) : 0;
  if (Tn + npad == 0) return LZ_OK;
  static const bool bulk = [] {
    const char* e = getenv("LZ_PACK_BULK");
    return e && atoi(e) != 0;
  }();
  const size_t pb_smem = (size_t)kPbWarps * kPbSlots * d * 2;
  if (bulk && pb_smem <= 200 * 1024 && d % 8 == 0) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(pack_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr = true;
    }
    return lzh::launch(pack_bulk_kernel, dim3(lzh::num_sms()), dim3(32 * kPbWarps), pb_smem,
                       (cudaStream_t)stream, 1, (const uint4*)x, Tn, d, k, row, prank, peers,
                       (uint4*)out, E, recv_m, recv_off, npad, ret_peers, ret_own, my_rank,
                       ret_row);
  }
  return lzh::launch(pack_kernel, dim3(row_grid(Tn + npad)), dim3(kRowThreads), 0,
                     (cudaStream_t)stream, 1, (const uint4*)x, Tn, d, k, row, prank, peers,
                     (uint4*)out, E, recv_m, recv_off, npad, ret_peers, ret_own, my_rank, ret_row);
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

extern "C" lz_status lz_pack_p2p_ret(const void* x, int Tn, int d, int k,
                                     const int32_t* dest_rank, const int32_t* dest_row,
                                     const unsigned long long* peers, void* own, int E,
                                     const int32_t* recv_m, const int32_t* recv_off,
                                     const unsigned long long* ret_peers, long long* ret_own,
                                     int my_rank, const int32_t* ret_row, void* stream) {
  if (!peers || !dest_rank || !ret_peers || !ret_own || my_rank < 0 || (Tn > 0 && !ret_row))
    return LZ_ERR_ARG;
  return pack_impl(x, Tn, d, k, dest_row, dest_rank, peers, own, E, recv_m, recv_off, stream,
                   ret_peers, ret_own, my_rank, ret_row);
}

static lz_status combine_impl(const void* y, const int32_t* row, const int32_t* prank,
                              const unsigned long long* peers, const float* w, int Tn, int d,
                              int k, void* out, void* stream) {
  if (Tn < 0 || d <= 0 || d % 8 || k < 1 || k > LZ_MAX_TOPK) return LZ_ERR_ARG;
  if (Tn == 0) return LZ_OK;
  if ((!y && !peers) || !row || !w || !out) return LZ_ERR_ARG;
  return lzh::launch(combine_kernel, dim3(row_grid(Tn)), dim3(kRowThreads), 0,
                     (cudaStream_t)stream, 1, (const uint4*)y, row, prank, peers, w, Tn, d, k,
                     (uint4*)out);
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
                                  const int32_t* recv_m, const int32_t* recv_off, void* stream,
                                  const int32_t* yrow = nullptr) {
  if (Tn < 0 || d <= 0 || d % 8 || k < 1 || k > LZ_MAX_TOPK || E < 0) return LZ_ERR_ARG;
  if (Tn > 0 && (!dout || (!y && !peers_y) || !row || !w || (!dy && !peers_dy) || !dw))
    return LZ_ERR_ARG;
  if (E > 0 && (!recv_m || !recv_off || !dy)) return LZ_ERR_ARG;
  const long npad = E > 0 ? pad_items(E, recv_m, recv_off, kPadAlign) : 0;
  if (Tn + npad == 0) return LZ_OK;
  return lzh::launch(combine_bwd_kernel, dim3(row_grid(Tn + npad)), dim3(kRowThreads), 0,
                     (cudaStream_t)stream, 1, (const uint4*)dout, (const uint4*)y, row, prank,
                     peers_y, peers_dy, w, Tn, d, k, (uint4*)dy, dw, E, recv_m, recv_off, npad,
                     yrow);
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

extern "C" lz_status lz_combine_bwd_p2p_ret(const void* dout, const void* y_ret,
                                            const int32_t* y_row,
                                            const unsigned long long* peers_dy,
                                            const int32_t* dest_rank, const int32_t* dest_row,
                                            const float* w, int Tn, int d, int k, float* dw,
                                            void* own_dy, int E, const int32_t* recv_m,
                                            const int32_t* recv_off, void* stream) {
  if (!y_ret || !peers_dy || !dest_rank || (Tn > 0 && !y_row)) return LZ_ERR_ARG;
  return combine_bwd_impl(dout, y_ret, dest_row, dest_rank, nullptr, peers_dy, w, Tn, d, k,
                          own_dy, dw, E, recv_m, recv_off, stream, y_row);
}

template <int KS, int ET>
static void d2_attr() {
  static bool done = false;   // one per instantiation
  if (!done) {
    cudaFuncSetAttribute(dispatch_bwd_reg<KS, ET>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kD2Smem);
    done = true;
  }
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
  if (d % 64 || E % 2) return LZ_ERR_UNSUPPORTED;
  const long dtasks = (Tn + kDT - 1) / kDT;
  const int nh = (d % 128 == 0) ? 2 : 1;   // column halves per 16-token tile (load balance)
  // persistent: as many blocks as are resident (4 per SM)
  long dgrid = (dtasks * nh + kD2Warps - 1) / kD2Warps;
  const long cap = (long)lzh::num_sms() * LZ_D2_BLOCKS;
  if (dgrid > cap) dgrid = cap;
#define LZ_DBWD(ks, et)                                                                      \
  (d2_attr<ks, et>(),                                                                        \
   lzh::launch(dispatch_bwd_reg<ks, et>, dim3((int)dgrid), dim3(32 * kD2Warps), kD2Smem,       \
               (cudaStream_t)stream, 1, (const uint4*)dxe, row, prank, peers, Tn, d, k, probs,  \
               idx, dw, (const __nv_bfloat16*)wg, E, renorm, (uint4*)dx, dlogits, nh))
  switch (E) {
    case 8: LZ_DBWD(1, 8); break;
    case 16: LZ_DBWD(1, 16); break;
    case 32: LZ_DBWD(2, 32); break;
    case 64: LZ_DBWD(4, 64); break;
    default:
      switch ((E + 15) / 16) {
        case 1: LZ_DBWD(1, 0); break;
        case 2: LZ_DBWD(2, 0); break;
        case 3: LZ_DBWD(3, 0); break;
        default: LZ_DBWD(4, 0); break;
      }
  }
#undef LZ_DBWD
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

// tensor-core path: d a multiple of 256 (whole warp column blocks); one block per SM
// per (column slice, expert group); else the FMA path with 2 blocks per SM
// tensor-core path: d a multiple of 128 (column slices of 128); ~8 blocks per SM over
// (token range, column slice, expert group); else the FMA path with 2 blocks per SM
static bool wgrad_tc(int d) { return d % kR2Cols == 0; }
static int wgrad_nblk(int Tn, int d, int E) {
  if (wgrad_tc(d)) {
    const int slices = (d / kR2Cols) * ((E + 15) / 16);
    int n = (LZ_R2_BLK * lzh::num_sms() + slices - 1) / slices;
    const int steps = (Tn + kR2Tok - 1) / kR2Tok;
    if (n > steps) n = steps;
    return n < 1 ? 1 : n;
  }
  int n = 2 * lzh::num_sms();
  long per = (Tn + n - 1) / n;
  if (per < 64) n = (Tn + 63) / 64;
  return n < 1 ? 1 : n;
}

extern "C" size_t lz_router_wgrad_ws_bytes(int Tn, int d, int E) {
  const size_t nblk = (size_t)wgrad_nblk(Tn, d, E);
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
  const int nblk = wgrad_nblk(Tn, d, E);
  float* part = (float*)ws;
  float* part_bias = part + (size_t)nblk * E * d;
  if (wgrad_tc(d)) {
    dim3 grid(nblk, d / kR2Cols, (E + 15) / 16);
    static bool attr2 = false;
    if (!attr2 && kR2Smem > 48 * 1024) {
      if (cudaFuncSetAttribute(router_wgrad_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kR2Smem) != cudaSuccess)
        return lzh::check_launch();
      attr2 = true;
    }
    lzh::launch(router_wgrad_tc2, grid, dim3(128), kR2Smem, s, 1, dlogits,
                (const __nv_bfloat16*)x, Tn, d, E, part, part_bias);
  } else {
    dim3 grid(nblk, (d + 1023) / 1024, (E + kWgE - 1) / kWgE);
    router_wgrad_partial<<<grid, 256, 0, s>>>(dlogits, (const __nv_bfloat16*)x, Tn, d, E, part,
                                              part_bias);
  }
  lz_status st = lzh::check_launch();
  if (st != LZ_OK) return st;
  const long n = (long)E * d;
  return lzh::launch(router_wgrad_reduce, dim3((int)((n + 31) / 32 + (E + 31) / 32)), dim3(256),
                     0, s, 1, (const float*)part, (const float*)part_bias, nblk, d, E, dwg, dbias);
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
