// gemm.cu -- K4/K5/K6: grouped expert GEMMs on 5th-gen tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel serves every FFN GEMM of the layer:
//   mode 0 (rows)  : per expert g, C[rows_g] = A[rows_g] . B_g      (fwd, dgrad)
//   mode 1 (wgrad) : per expert g, C_g = A[rows_g]^T . B[rows_g]    (variable-K weight grad)
// Tile 128 x 256 x 64 (bf16), UMMA 128x256x16 (kind::f16, fp32 accumulate in TMEM),
// 4-stage TMA -> smem ring (128B swizzle), double-buffered TMEM accumulator
// (2 x 256 columns) so the epilogue of tile i overlaps the main loop of tile i+1.
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one lane issues tcgen05.mma)
//   warps 2..9  epilogue: tcgen05.ld 32x32b -> fused activation -> bf16 -> smem -> TMA store
// The reference has no FFN code; semantics follow PAPER.md:143
// (one weight copy per (expert, rank); R[e][j] > 1 only scales capacity).
#include <cuda.h>  // CUtensorMap (header only; the encoder is fetched at run time)

#include <stdlib.h>

#include <type_traits>

#include "common.cuh"

namespace lz {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 64;  // per-CTA rows, tile columns, k block
constexpr int kEpiWarps = 8;                       // 2 per TMEM lane quadrant (column halves)
constexpr int kThreads = 64 + 32 * kEpiWarps;      // producer, MMA, epilogue warps
constexpr int kAccCols = BN;              // fp32 accumulator columns per buffer
constexpr int kTmemCols = 2 * kAccCols;   // 512
constexpr int kMaxGroups = 128;
// epilogue staging: each epilogue warp owns 32 rows; chunks of 32 columns (64 B rows,
// 64B-swizzled, 2 KB), double-buffered, feed the TMA stores of the outputs (aux streams
// go straight between registers and global memory, see aux_block)
constexpr int kEpiCols = 32;
constexpr int kEpiBuf = 32 * kEpiCols * 2;          // 2 KB
constexpr int kBarBytes = 256;
constexpr int kSchedSlots = 4;   // dynamic scheduler queue depth
constexpr int kTabBytes = 3 * (kMaxGroups + 1) * 4;  // s_off, s_pref, s_perm

// CG = 1: one CTA per 128 x 256 tile (UMMA 128x256x16, cta_group::1), 3-4 stages x 48 KB.
// CG = 2: a CTA pair per 256 x 256 tile (UMMA 256x256x16, cta_group::2): each CTA stages
//         its 128 rows of A and half (128 columns) of B -> 32 KB/stage, 5-6 stages; the
//         leader CTA issues the MMAs for both, halving per-SM smem operand traffic.
// AUX: the epilogue has an aux stream (GELU/dGELU/SwiGLU/dSwiGLU; compile-time split so
// the plain-store variant carries none of the activation code).  Aux streams bypass
// shared memory (aux_block), so every variant stages only its outputs: 2 x 2 KB per
// epilogue warp, leaving room for 6 (CTA pair) / 4 (single CTA) operand stages.
// NS = 2 (CTA pair, weight-gradient GEMMs): a 256 x 512 tile as two 256-column UMMAs per
// k step sharing the A stage -- the A operand is read from L2 once per 512 output columns
// (L2 -> SM operand traffic -25 %).  Its 512 accumulator columns fill TMEM, so there is one
// accumulator (the epilogue of tile i is not overlapped with the main loop of tile i + 1;
// with the weight gradients' long K that costs ~2 % and the GEMMs are L2-bound).
template <int CG, bool AUX, int NS = 1>
struct Cfg {
  static constexpr int kEpiWarpBytes = 2 * kEpiBuf;
  static constexpr int kEpiBytes = kEpiWarps * kEpiWarpBytes;
  static constexpr int kTileN = BN * NS;                 // output columns per tile
  static constexpr int kBRows = BN / CG;                 // B rows (n) per sub-tile per CTA
  static constexpr int kATileBytes = BM * BK * 2;        // 16 KB
  static constexpr int kBSubBytes = kBRows * BK * 2;     // 32 KB / 16 KB per sub-tile
  static constexpr int kBTileBytes = NS * kBSubBytes;
  static constexpr int kStageBytes = kATileBytes + kBTileBytes;
  static constexpr int kStages = CG == 1 ? 4 : (NS == 1 ? 6 : 4);
  static constexpr int kNAcc = NS == 1 ? 2 : 1;          // TMEM accumulator buffers
  static constexpr int kTilesBytes = kStages * kStageBytes;
  static constexpr int kTileM = BM * CG;                 // rows per (pair) tile
  static constexpr int kSmemBytes = 1024 + kTilesBytes + kEpiBytes + kBarBytes + kTabBytes;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
#ifndef LZ_NO_WATCHDOG
  // a pipeline bug must fail loudly, not hang the GPU: after ~10 s of waiting record it in
  // the control block and give up (the kernel then runs to its end and the host discards
  // the step); without a control block, trap
  const long long t0 = clock64();
#endif
  do {
    // suspend-time hint: the waiting warp sleeps in the barrier unit until the phase
    // completes (or ~0.1 ms passes) instead of re-polling -- fewer issue slots and less
    // power burnt by the idle roles of the persistent kernel
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(100000)
        : "memory");
#ifndef LZ_NO_WATCHDOG
    if (!done) {
      const long long dt = clock64() - t0;
      if (dt > (1ll << 24)) {   // slow path only (~8 ms): a healthy wait never gets here
        lz_ctl* c = g_ctl;
        if (c && ld_sys_s32(&c->watchdog)) return;   // another wait already gave up
        if (dt > 20000000000ll) {
          if (!c) __trap();
          st_sys_s32(&c->watchdog, 1);
          return;
        }
      }
    }
#endif
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 2-CTA variant: the transaction bytes are credited to the leader CTA's barrier (the
// CTA-rank bit 24 of the shared::cluster address cleared), data lands in local smem.
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
template <int CG>
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                         int c1) {
  if (CG == 1) tma_load_2d(dst, map, bar, c0, c1);
  else tma_load_2d_cg2(dst, map, bar, c0, c1);
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same smem offset in CTA `cta` of the cluster.  Relaxed:
// it only signals "TMEM accumulator drained" -- the tcgen05.ld data is already in
// registers (tcgen05.wait::ld), so no memory needs releasing, and a release.cluster
// arrive costs MEMBAR.ALL.GPU + ERRBAR per epilogue warp per tile (ncu r01c).
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
// the accumulator-empty barrier lives in the leader CTA (rank 0), which issues the MMAs
__device__ __forceinline__ void tmem_release(uint64_t* bar, int cg) {
  if (cg == 1 || cluster_ctarank() == 0) mbar_arrive(bar);
  else mbar_arrive_cluster(bar, 0);
}
template <int CG>
__device__ __forceinline__ void tc_commit_cg(uint64_t* bar) {
  if (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
  } else {
    // arrive on the same barrier in both CTAs of the pair
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tc_mma_cg(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
  if (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  }
}

// Warp-uniform issue: the whole MMA warp runs the issue loop (uniform control flow, so
// descriptors and stage indices live in uniform registers) and elect.sync picks the one
// lane that issues, inside the same asm block.  Issuing from `if (lane == 0)` instead
// made ptxas wrap every tcgen05.mma in an ELECT / R2UR.BROADCAST / BRA.U.ANY waterfall
// loop (~95 instructions per 64-deep k block), and with two heavy-epilogue warps on the
// same SMSP the issuer fell behind the tensor pipe (ncu r01e: GELU GEMM 62 % active).
template <int CG>
__device__ __forceinline__ void tc_mma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accum) {
  if (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  }
}
template <int CG>
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  if (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;\n\t}" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  }
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// byte offset of 16-byte piece q of row r inside a 64B-swizzled [32 x 64 B] staging tile
__device__ __forceinline__ int stg_off(int r, int q) { return r * 64 + ((q ^ ((r >> 1) & 3)) << 4); }
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

// UMMA shared-memory descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), layout type [61,64) (2 = 128B swizzle).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t make_idesc(int a_mn, int b_mn, int m = BM) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// tanh-approximate GELU ("gelu_new", GPT-2 MLP) and its derivative.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kS2PI = 0.7978845608028654f;
constexpr float kGC = 0.044715f;
// The forward GELU epilogue stores gelu'(h) (not h) as the backward's aux stream, so the
// dGELU epilogue is a plain multiply (no MUFU in the backward GEMM epilogue).
// Packed fp32x2 arithmetic (sm_100 FFMA2 / FMUL2): half the issue slots of scalar FP32
// for the epilogue math, which is issue/latency-bound next to the tensor pipe.
__device__ __forceinline__ unsigned long long f2_u64(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 u64_f2(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_u64(a)), "l"(f2_u64(b)), "l"(f2_u64(c)));
  return u64_f2(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(r);
}
__device__ __forceinline__ float2 splat2(float v) { return make_float2(v, v); }
// gelu and gelu' of two values, 10 packed ops + 2 tanh:  s = (1 + t) / 2,  gelu = x s,
// gelu' = s + x (-2 q) s (s - 1)  with  q = du/dx = c0 (1 + 3 kGC x^2)  (1 - t^2 = 4 s (1 - s))
__device__ __forceinline__ void gelu_and_grad2(float2 x, float2& y, float2& dy) {
  constexpr float c0 = kS2PI, c1 = kS2PI * kGC;
  const float2 x2 = mul2(x, x);
  const float2 u = mul2(x, fma2(x2, splat2(c1), splat2(c0)));
  const float2 t = make_float2(tanh_fast(u.x), tanh_fast(u.y));
  const float2 sv = fma2(t, splat2(0.5f), splat2(0.5f));
  const float2 z = fma2(t, splat2(0.5f), splat2(-0.5f));
  const float2 wn = mul2(x, fma2(x2, splat2(-6.f * c1), splat2(-2.f * c0)));
  y = mul2(x, sv);
  dy = fma2(wn, mul2(sv, z), sv);
}

struct Params {
  int mode;         // 0 rows, 1 wgrad
  int c_grp_rows;   // mode 1: rows between consecutive groups' C blocks (>= M)
  int c_row_off;    // mode 1: row offset of group 0's C block
  int G;            // groups
  int M, N, K;      // mode 0: N, K used; mode 1: M, N
  const int32_t* off;
  int epilogue;
  __nv_bfloat16* C;
  __nv_bfloat16* aux;
  // scatter epilogue (store variant, mode 0): output row r goes to rank (ret_map[r] >> 32)
  // at row (ret_map[r] & 0xffffffff) of its buffer ret_peers[rank] (row length N); -1 = pad
  const long long* ret_map;
  const unsigned long long* ret_peers;
  // arrival-ordered row GEMM (mode 0, multi-GPU): self_rows[2g], [2g+1] = rows of group g
  // this rank sent to itself; tiles fully inside them run first, every other tile waits
  // until flags[0..n_flags) (written by the senders after their dispatch) reach *epoch
  const int32_t* self_rows;
  const int* flags;
  int n_flags;
  const int* epoch;
  // L2-aware rasterisation of the row GEMMs (mode 0): the expert's weight slices (K x 256
  // per n-block) that concurrently running tiles re-read are visited in chunks of at most
  // this many bytes, so a chunk stays L2-resident while the token rows stream (cfg3
  // W1|W3 is 235 MB per expert: n-fastest order re-read it from DRAM for every m-block,
  // 27 GB per launch)
  long long l2_chunk_bytes;
  // dynamic tile scheduler (non-null): [0] next tile, [1] units done -- the leader CTA of
  // each unit fetches tiles with an atomic add and hands them to its roles (and to the
  // peer CTA) through a shared-memory queue; the last unit resets both counters
  int* tile_ctr;
};

// Tile `local` of an (n_outer x n_inner) grid, ordered: for each chunk of `c` inner
// blocks, for each outer block, for each inner block of the chunk.  c >= n_inner is the
// plain inner-fastest order.
__device__ __forceinline__ void chunked_raster(int local, int n_outer, int n_inner, int c, int& o,
                                               int& i) {
  if (c >= n_inner) {
    o = local / n_inner;
    i = local - o * n_inner;
    return;
  }
  const int per_chunk = n_outer * c;
  const int ch = local / per_chunk;
  const int rem = local - ch * per_chunk;
  const int cw = min(c, n_inner - ch * c);
  o = rem / cw;
  i = ch * c + (rem - o * cw);
}
__device__ __forceinline__ int chunk_blocks(long long budget, long long slice_bytes, int n) {
  long long c = slice_bytes > 0 ? budget / slice_bytes : n;
  return (int)(c < 1 ? 1 : (c > n ? n : c));
}

// Per-rank tensor maps of the scatter GEMM's return buffers ([rows, N] bf16 each): a
// 32-row chunk whose rows return to consecutive rows of one rank (the common case: the
// dispatch lays every (owner, expert) segment out contiguously on the source) is one TMA
// store into that rank's buffer, over NVLink for remote ranks.
constexpr int kMaxRetPeers = 8;
struct RetMaps {
  CUtensorMap m[kMaxRetPeers];
  int n;
};

// A tile load (128 x 64) for the current stage
template <int A_MN, int CG>
__device__ __forceinline__ void load_a(const CUtensorMap* map, uint8_t* dst, uint64_t* bar,
                                       int row_or_k, int m0, int k0) {
  if (A_MN == 0) {
    tma_load<CG>(dst, map, bar, k0, row_or_k);  // K-major: (k, row), 128 rows
  } else {
    // MN-major: two 64-wide M boxes of 64 k-rows
    tma_load<CG>(dst, map, bar, m0, row_or_k);
    tma_load<CG>(dst + 8192, map, bar, m0 + 64, row_or_k);
  }
}
template <int B_MN, int CG>
__device__ __forceinline__ void load_b(const CUtensorMap* map, uint8_t* dst, uint64_t* bar,
                                       int n_row, int n0, int k_row, int k0) {
  if (B_MN == 0) {
    tma_load<CG>(dst, map, bar, k0, n_row);  // K-major (k, n-row), BN/CG rows
  } else {
#pragma unroll
    for (int q = 0; q < 4 / CG; ++q) tma_load<CG>(dst + 8192 * q, map, bar, n0 + 64 * q, k_row);
  }
}

struct TileInfo {
  int g, mb, nb, nk;
  bool remote;   // may contain rows dispatched by other ranks (arrival-ordered GEMM)
};

template <int CG>
__host__ __device__ constexpr int C_TILE_M() { return BM * CG; }

template <int CG, int NS = 1>
__device__ __forceinline__ TileInfo decode_tile(const Params& p, const int32_t* s_pref,
                                                const int32_t* s_off, const int32_t* s_perm,
                                                int total0, int tile) {
  // (tiles are TileM x BN*NS; mb counts TileM blocks, nb tile-wide column blocks).
  // mode 1: tiles numbered over the groups in s_perm order (descending K).
  // mode 0: class-0 tiles (fully inside a group's self rows, count s_perm[g] >> 16 m-blocks
  //         from m-block s_perm[g] & 0xffff) come first, then the class-1 rest in group
  //         order (prefix s_pref); without self rows class 0 is empty.
  const int nbn = p.N / (BN * NS);
  TileInfo t;
  t.remote = false;
  // mode 0: B slices (K x 256 weights per n-block) are the re-read operand
  const int cb0 =
      p.mode == 0 ? chunk_blocks(p.l2_chunk_bytes, (long long)p.K * BN * NS * 2, nbn) : 0;
  if (p.mode == 0 && tile < total0) {
    int acc = 0, g = 0;
    for (; g < p.G - 1; ++g) {
      const int n0 = (s_perm[g] >> 16) * nbn;
      if (tile < acc + n0) break;
      acc += n0;
    }
    const int local = tile - acc;
    int mbl, nb;
    chunked_raster(local, s_perm[g] >> 16, nbn, cb0, mbl, nb);
    t.g = g;
    t.mb = (s_perm[g] & 0xffff) + mbl;
    t.nb = nb;
    t.nk = p.K / BK;
    return t;
  }
  const int t1 = p.mode == 0 ? tile - total0 : tile;
  int lo = 0, hi = p.G - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_pref[mid] <= t1) lo = mid;
    else hi = mid - 1;
  }
  const int local = t1 - s_pref[lo];
  if (p.mode == 0) {
    t.g = lo;
    const int c0 = s_perm[lo] >> 16, mlo = s_perm[lo] & 0xffff;
    const int nmb1 = (s_pref[lo + 1] - s_pref[lo]) / nbn;
    int mbl, nb;
    chunked_raster(local, nmb1, nbn, cb0, mbl, nb);
    t.nb = nb;
    t.mb = mbl < mlo ? mbl : mbl + c0;
    t.nk = p.K / BK;
    t.remote = p.self_rows != nullptr;
  } else {
    // weight gradient: raster along the smaller output dimension so the concurrently
    // running tiles share the operand slices of the larger one (cfg3 dW2 = dY^T A with
    // M = 4096, N = 14336: N-fastest order streamed A's 256-column slices from DRAM once
    // per m-block).  No chunking here: the slices along the smaller dimension are the
    // few ones, and chunking them re-reads the many ones (cfg3 dW1: 2.7x the 1.9 GB dH)
    const int nbm = p.M / C_TILE_M<CG>();
    t.g = s_perm[lo];
    const int rows_g = s_off[t.g + 1] - s_off[t.g];
    if (nbm <= nbn) {
      chunked_raster(local, nbn, nbm, nbm, t.nb, t.mb);
    } else {
      chunked_raster(local, nbm, nbn, nbn, t.mb, t.nb);
    }
    t.nk = rows_g / BK;
  }
  return t;
}

// Producer side of the arrival-ordered GEMM: wait until every sender has signalled this
// step's dispatch into our receive buffer (release stores by lz_signal_peers), then make
// the remote rows visible to the TMA (async proxy).
// Bounded (lz_ctl): a sender that never signals -- a rank lost mid-step -- makes the wait
// give up after the control block's timeout (or at once when the host raises abort); the
// GEMM then runs on whatever rows are present and the host discards the step.
__device__ __forceinline__ void wait_arrivals(const Params& p) {
  int want;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(want) : "l"(p.epoch) : "memory");
  long long deadline = 0;
  for (int i = 0; i < p.n_flags; ++i) {
    int v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p.flags + i) : "memory");
      if (v - want >= 0) break;
      if (peer_wait_give_up(deadline)) {
        i = p.n_flags;
        break;
      }
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Private "epilogue-native" layout of the aux streams (GELU: gelu'(h); SwiGLU: S | Q),
// written by a forward epilogue and read only by the matching backward epilogue: 32 x 32
// blocks, block (r/32, c/32) at ((r/32) * (W/32) + c/32) * 1024 elements (W = aux width);
// inside a block, element (row l, col 8q + i) sits at q * 256 + l * 8 + i -- so
// instruction q of a warp whose lane l owns row l reads/writes 512 contiguous bytes, with
// no shared-memory staging.  Same byte size as row-major [rows, W].
__device__ __forceinline__ uint4* aux_block(const Params& p, int width, int row0, int col) {
  return reinterpret_cast<uint4*>(p.aux) +
         ((size_t)(row0 >> 5) * (width >> 5) + (col >> 5)) * 128;
}

// Static persistent schedule: wave w hands tile w*nunits + slot to unit `unit`, with the
// slot order reversed on odd waves ("snake").  With tiles numbered in descending cost
// (weight-gradient groups sorted by their K = rows) this is the LPT-style balance a
// round-robin over expert-major tiles lacks (ncu r01c: wgrad 80 % vs 88 % tensor-active).
__device__ __forceinline__ int sched_tile(int w, int unit, int nunits) {
  return w * nunits + ((w & 1) ? nunits - 1 - unit : unit);
}

// SwiGLU epilogues (Mixtral experts).  W1|W3 are interleaved in blocks of 128 output
// rows, so one 256-wide N tile holds the gate (cols 0..127) and up (cols 128..255)
// projections of the same 128 hidden units.
//   SWIGLU : C[rows, N/2] = silu(g) * u at hidden column nb*128 + j; AUX [rows, N] keeps
//            the backward's factors S = silu(g) (gate column), Q = u silu'(g) (up column)
//   DSWIGLU: GEMM output dA[rows, N] (N = d_ff, hidden units); reads S, Q from AUX
//            [rows, 2N] and writes dH = [dG | dU] = [dA Q | dA S] into C[rows, 2N]
// AUX uses the private blocked layout (aux_block), accessed straight from registers.
// Each epilogue warp owns 32 rows and one half of the tile's hidden units; the output
// staging is double-buffered (2 x 2 KB per warp).
__device__ __forceinline__ void swiglu_epilogue(const Params& p, bool fwd, const TileInfo& t,
                                             int row0, int half, int lane, uint32_t tbase,
                                             uint64_t* tfull, uint32_t acc_phase,
                                             uint64_t* tempty, uint8_t* wbuf,
                                             const CUtensorMap* map_c, int cg) {
  const uint32_t s_out = smem_u32(wbuf);
  const int nchunks = fwd ? 2 : 4;  // 64 hidden units (fwd) / 128 hidden units (bwd) per warp
  const int auxw = fwd ? p.N : 2 * p.N;
  auto cols = [&](int c, int& gcol, int& ucol, int& hid) {
    if (fwd) {
      hid = t.nb * (BN / 2) + half * 64 + c * 32;              // Act column
      gcol = t.nb * BN + half * 64 + c * 32;                   // gate column in H
      ucol = gcol + BN / 2;
    } else {
      const int n0 = t.nb * BN + half * 128 + c * 32;          // hidden unit
      hid = n0;
      gcol = (n0 / 128) * 256 + (n0 % 128);
      ucol = gcol + 128;
    }
  };
  uint4 sn[4], qn[4];  // backward: next chunk's S and Q (in flight during this chunk)
  if (!fwd) {
    int g, u, h;
    cols(0, g, u, h);
    const uint4* ps = aux_block(p, auxw, row0, g) + lane;
    const uint4* pq = aux_block(p, auxw, row0, u) + lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      sn[q] = ld_nc_v4(ps + q * 32);
      qn[q] = ld_nc_v4(pq + q * 32);
    }
  }
  mbar_wait(tfull, acc_phase);
  tc_fence_after();
  for (int c = 0; c < nchunks; ++c) {
    int gcol, ucol, hid;
    cols(c, gcol, ucol, hid);
    uint32_t va[32], vb[32];
    if (fwd) {
      tmem_ld32(tbase + half * 64 + c * 32, va);           // gate
      tmem_ld32(tbase + BN / 2 + half * 64 + c * 32, vb);  // up
    } else {
      tmem_ld32(tbase + half * 128 + c * 32, va);          // dA
    }
    if (t.nk == 0) {
#pragma unroll
      for (int q = 0; q < 32; ++q) va[q] = vb[q] = 0u;
    }
    if (c == nchunks - 1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) tmem_release(tempty, cg);
    }
    if (fwd) {
      // out buffer c & 1: the store issued two chunks ago (previous tile) must be done
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
      uint4* ps = aux_block(p, auxw, row0, gcol) + lane;
      uint4* pq = aux_block(p, auxw, row0, ucol) + lane;
      const uint32_t so = s_out + (c & 1) * kEpiBuf;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float a[8], sv[8], qv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          // packed: sg = (1 + tanh(g/2)) / 2, S = g sg, act = S u, Q = u sg (1 + g (1 - sg))
          const int j = 8 * q + i;
          const float2 g2 = make_float2(__uint_as_float(va[j]), __uint_as_float(va[j + 1]));
          const float2 u2 = make_float2(__uint_as_float(vb[j]), __uint_as_float(vb[j + 1]));
          const float2 h2 = mul2(g2, splat2(0.5f));
          const float2 t2 = make_float2(tanh_fast(h2.x), tanh_fast(h2.y));
          const float2 sg = fma2(t2, splat2(0.5f), splat2(0.5f));
          const float2 om = fma2(t2, splat2(-0.5f), splat2(0.5f));
          const float2 sl = mul2(g2, sg);
          const float2 a2 = mul2(sl, u2);
          const float2 q2 = mul2(mul2(u2, sg), fma2(g2, om, splat2(1.f)));
          a[i] = a2.x;
          a[i + 1] = a2.y;
          sv[i] = sl.x;
          sv[i + 1] = sl.y;
          qv[i] = q2.x;
          qv[i + 1] = q2.y;
        }
        st_v4(ps + q * 32, f32_to_bf16x8(sv));
        st_v4(pq + q * 32, f32_to_bf16x8(qv));
        st_shared_v4(so + stg_off(lane, q), f32_to_bf16x8(a));
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map_c, wbuf + (c & 1) * kEpiBuf, hid, row0);
        bulk_commit();
      }
    } else {
      uint4 sc[4], qc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        sc[q] = sn[q];
        qc[q] = qn[q];
      }
      if (c + 1 < nchunks) {
        int g2, u2, h2;
        cols(c + 1, g2, u2, h2);
        const uint4* ps = aux_block(p, auxw, row0, g2) + lane;
        const uint4* pq = aux_block(p, auxw, row0, u2) + lane;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          sn[q] = ld_nc_v4(ps + q * 32);
          qn[q] = ld_nc_v4(pq + q * 32);
        }
      }
      // both staging buffers are rewritten: the previous chunk's two stores must be done
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float sf[8], qf[8], dg[8], du[8];
        bf16x8_to_f32(sc[q], sf);
        bf16x8_to_f32(qc[q], qf);
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float2 da = make_float2(__uint_as_float(va[8 * q + i]),
                                        __uint_as_float(va[8 * q + i + 1]));
          const float2 x = mul2(da, make_float2(qf[i], qf[i + 1]));
          const float2 y = mul2(da, make_float2(sf[i], sf[i + 1]));
          dg[i] = x.x;
          dg[i + 1] = x.y;
          du[i] = y.x;
          du[i + 1] = y.y;
        }
        st_shared_v4(s_out + stg_off(lane, q), f32_to_bf16x8(dg));
        st_shared_v4(s_out + kEpiBuf + stg_off(lane, q), f32_to_bf16x8(du));
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map_c, wbuf, gcol, row0);
        tma_store_2d(map_c, wbuf + kEpiBuf, ucol, row0);
        bulk_commit();
      }
    }
  }
}

template <int A_MN, int B_MN, int CG, bool AUX, int NS>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_c,
                        const __grid_constant__ CUtensorMap map_x, const Params p,
                        const __grid_constant__ RetMaps rmaps) {
  using C = Cfg<CG, AUX, NS>;
  static_assert(NS == 1 || (CG == 2 && !AUX), "256 x 512 tiles: CTA pair, store epilogue");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* s_tiles = smem;
  uint8_t* s_epi = smem + C::kTilesBytes;
  uint64_t* full_bar = (uint64_t*)(s_epi + C::kEpiBytes);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tfull_bar = empty_bar + C::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* sched_full = tempty_bar + 2;             // [kSchedSlots] tile id published
  uint64_t* sched_empty = sched_full + kSchedSlots;   // [kSchedSlots] all roles read it
  int32_t* s_sched = (int32_t*)(sched_empty + kSchedSlots);   // [kSchedSlots] tile ids
  uint32_t* s_tmem = (uint32_t*)(s_sched + kSchedSlots);
  int32_t* s_total0 = (int32_t*)(s_tmem + 1);   // class-0 tile count (mode 0)
  int32_t* s_off = (int32_t*)((uint8_t*)full_bar + kBarBytes);
  int32_t* s_pref = s_off + kMaxGroups + 1;

  pdl_launch_dependents();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t cta = CG == 1 ? 0u : cluster_ctarank();
  const bool leader = cta == 0;
  const int unit = CG == 1 ? blockIdx.x : (blockIdx.x >> 1);   // tile-processing unit
  const int nunits = CG == 1 ? gridDim.x : (gridDim.x >> 1);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], kEpiWarps * CG);  // one arrival per epilogue warp of each CTA
    }
    for (int s = 0; s < kSchedSlots; ++s) {
      mbar_init(&sched_full[s], 1);
      // read by: the MMA warp and every epilogue warp of the leader, the peer's producer and
      // every epilogue warp of the peer
      mbar_init(&sched_empty[s], CG == 1 ? 1 + kEpiWarps : 2 + 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_c) : "memory");
    if (p.epilogue != LZ_EPI_STORE) asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
  }
  if (warp == 1) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(s_tmem)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(s_tmem)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  // barrier init, tensor-map prefetch and TMEM allocation above overlap the predecessor's
  // tail (PDL); the device offsets and every operand only after the wait
  pdl_wait();
  // group table -> tile prefix (every CTA computes it; G <= kMaxGroups).  Weight-gradient
  // groups are visited in descending K (tile cost); row GEMM tiles all cost the same.
  int32_t* s_perm = s_pref + kMaxGroups + 1;
  for (int g = threadIdx.x; g <= p.G; g += blockDim.x) s_off[g] = p.off[g];
  __syncthreads();
  for (int g = threadIdx.x; g < p.G; g += blockDim.x) {
    if (p.mode == 1) {
      const int kg = s_off[g + 1] - s_off[g];
      int rank = 0;
      for (int h = 0; h < p.G; ++h) {
        const int kh = s_off[h + 1] - s_off[h];
        rank += (kh > kg) || (kh == kg && h < g);
      }
      s_perm[rank] = g;
    } else {
      // self-row m-block window of group g: (count << 16) | first m-block
      int c0 = 0, mlo = 0;
      if (p.self_rows) {
        const int base = s_off[g];
        const int lo = p.self_rows[2 * g] - base, hi = p.self_rows[2 * g + 1] - base;
        mlo = (lo + C::kTileM - 1) / C::kTileM;
        const int mhi = hi / C::kTileM;
        c0 = mhi > mlo ? mhi - mlo : 0;
        if (c0 == 0) mlo = 0;
      }
      s_perm[g] = (c0 << 16) | mlo;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0, acc0 = 0;
    const int nbn = p.N / C::kTileN;
    for (int i = 0; i < p.G; ++i) {
      s_pref[i] = acc;
      if (p.mode == 0) {
        const int c0 = s_perm[i] >> 16;
        acc += ((s_off[i + 1] - s_off[i]) / C::kTileM - c0) * nbn;
        acc0 += c0 * nbn;
      } else {
        acc += (p.M / C::kTileM) * nbn;
      }
    }
    s_pref[p.G] = acc;
    *s_total0 = acc0;
  }
  tc_fence_before();
  if (CG == 1) __syncthreads();
  else cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  const int total0 = *s_total0;
  const int total = s_pref[p.G] + total0;
  const bool dyn = p.tile_ctr != nullptr;
  // Tile feed of one role.  Static: the snake schedule.  Dynamic: the leader CTA's producer
  // fetches with an atomic add and publishes into the queue (also into the peer CTA's);
  // every other role reads the queue and releases the slot to the leader's producer.
  int f_w = 0, f_q = 0, f_pend = -1, f_ahead = -1;
  uint32_t f_ph = 0;
  // (publisher) publish tile t into queue slot f_q of both CTAs of the unit
  auto publish = [&](int t) {
    mbar_wait(&sched_empty[f_q], f_ph ^ 1);
    s_sched[f_q] = t;
    if (CG == 2) {
      asm volatile(
          "{\n\t.reg .b32 ra, rb;\n\t"
          "mapa.shared::cluster.u32 ra, %0, 1;\n\t"
          "st.shared::cluster.s32 [ra], %2;\n\t"
          "mapa.shared::cluster.u32 rb, %1, 1;\n\t"
          "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [rb];\n\t}" ::"r"(
              smem_u32(&s_sched[f_q])),
          "r"(smem_u32(&sched_full[f_q])), "r"(t)
          : "memory");
    }
    mbar_arrive(&sched_full[f_q]);
    if (++f_q == kSchedSlots) {
      f_q = 0;
      f_ph ^= 1;
    }
  };
  // (publisher) the next fetched tile; the atomic for the one after is already in flight
  auto fetch = [&]() -> int {
    const int t = f_pend;
    f_pend = atomicAdd(p.tile_ctr, 1);
    return t < total ? t : total;
  };
  auto next_tile = [&](bool publisher) -> int {
    if (!dyn) {
      const int t = sched_tile(f_w, unit, nunits);
      ++f_w;
      return t;
    }
    int tile;
    if (publisher) {
      // the queue runs one tile ahead of the publisher's own loads, so the peer CTA and the
      // MMA / epilogue roles already know tile i+1 when tile i starts
      if (f_ahead < 0) {
        f_pend = atomicAdd(p.tile_ctr, 1);
        f_ahead = fetch();
        publish(f_ahead);
      }
      tile = f_ahead;
      if (tile < total) {
        f_ahead = fetch();
        publish(f_ahead);
      }
      return tile;
    } else {
      mbar_wait(&sched_full[f_q], f_ph);
      tile = *reinterpret_cast<volatile int32_t*>(&s_sched[f_q]);
      // the producer role runs on one lane, the MMA and epilogue roles on whole warps:
      // one release per role instance, after all of its lanes have read the slot
      const unsigned am = __activemask();
      __syncwarp(am);
      if (lane == __ffs(am) - 1) {
        if (CG == 1 || leader) {
          mbar_arrive(&sched_empty[f_q]);
        } else {
          asm volatile(
              "{\n\t.reg .b32 ra;\n\t"
              "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
              "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(
                  smem_u32(&sched_empty[f_q]))
              : "memory");
        }
      }
    }
    if (++f_q == kSchedSlots) {
      f_q = 0;
      f_ph ^= 1;
    }
    return tile;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs of a pair load their halves) =====
      int stage = 0;
      uint32_t phase = 0;
      bool arrived = p.flags == nullptr;
      for (int tile = next_tile(leader); tile < total; tile = next_tile(leader)) {
        const TileInfo t = decode_tile<CG, NS>(p, s_pref, s_off, s_perm, total0, tile);
        if (t.remote && !arrived) {   // first tile with rows from other ranks
          wait_arrivals(p);
          arrived = true;
        }
        for (int kb = 0; kb < t.nk; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = s_tiles + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kATileBytes;
          if (leader) mbar_expect_tx(&full_bar[stage], CG * C::kStageBytes);
          if (p.mode == 0) {
            const int row = s_off[t.g] + t.mb * C::kTileM + cta * BM;
            load_a<A_MN, CG>(&map_a, sa, &full_bar[stage], row, 0, kb * BK);
#pragma unroll
            for (int j = 0; j < NS; ++j) {
              const int n0 = t.nb * C::kTileN + j * BN + cta * C::kBRows;
              load_b<B_MN, CG>(&map_b, sb + j * C::kBSubBytes, &full_bar[stage], t.g * p.N + n0,
                               n0, t.g * p.K + kb * BK, kb * BK);
            }
          } else {
            const int krow = s_off[t.g] + kb * BK;
            load_a<A_MN, CG>(&map_a, sa, &full_bar[stage], krow, t.mb * C::kTileM + cta * BM, 0);
#pragma unroll
            for (int j = 0; j < NS; ++j)
              load_b<B_MN, CG>(&map_b, sb + j * C::kBSubBytes, &full_bar[stage], 0,
                               t.nb * C::kTileN + j * BN + cta * C::kBRows, krow, 0);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (dyn && leader) {
        // this unit fetched its end marker: the last unit to get here resets the counters
        // for the next launch (no unit fetches after its own end marker)
        __threadfence();
        if (atomicAdd(p.tile_ctr + 1, 1) == nunits - 1) {
          p.tile_ctr[0] = 0;
          p.tile_ctr[1] = 0;
          __threadfence();
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer (leader CTA issues for the pair; whole warp, one elected lane) ====
      constexpr uint32_t idesc = make_idesc(A_MN, B_MN, BM * CG);
      // descriptors of stage 0; stage s / k step k are plain adds to the start-address
      // field (smem addresses < 256 KB: (addr >> 4) never carries out of its 14 bits)
      const uint32_t sa0 = smem_u32(s_tiles);
      const uint64_t da0 = A_MN ? make_desc(sa0, 8192, 1024) : make_desc(sa0, 16, 1024);
      const uint64_t db0 = B_MN ? make_desc(sa0 + C::kATileBytes, 8192, 1024)
                                : make_desc(sa0 + C::kATileBytes, 16, 1024);
      // K-major: +32 B per 16-element k step inside the 128 B swizzle atom
      // MN-major: +2 x (8 rows x 128 B) per 16 k rows; atoms along MN are 8 KB apart
      constexpr uint64_t kStepA = A_MN ? (2048 >> 4) : (32 >> 4);
      constexpr uint64_t kStepB = B_MN ? (2048 >> 4) : (32 >> 4);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = next_tile(false); tile < total; tile = next_tile(false)) {
        const TileInfo t = decode_tile<CG, NS>(p, s_pref, s_off, s_perm, total0, tile);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        for (int kb = 0; kb < t.nk; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t soff = (uint64_t)(stage * (C::kStageBytes >> 4));
          const uint64_t ad = da0 + soff, bd = db0 + soff;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
#pragma unroll
            for (int j = 0; j < NS; ++j)   // sub-tile j: accumulator columns [256 j, +256)
              tc_mma_elect<CG>(d_tmem + j * BN, ad + k * kStepA,
                               bd + (uint64_t)(j * (C::kBSubBytes >> 4)) + k * kStepB, idesc,
                               (kb | k) != 0);
          tc_commit_elect<CG>(&empty_bar[stage]);  // frees the smem slot(s) when the MMAs retire
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_elect<CG>(&tfull_bar[acc]);  // accumulator ready for the epilogue(s)
        if (++acc == C::kNAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===== epilogue warps 2..5: TMEM -> regs -> activation -> swizzled smem -> TMA store
    const int quad = warp & 3;          // TMEM lane quadrant this warp may access
    const int ew = warp - 2;            // epilogue warp index
    const int half = ew >> 2;           // column half of the tile this warp owns
    uint8_t* wbuf = s_epi + ew * C::kEpiWarpBytes;
    const uint32_t out_s = smem_u32(wbuf);                 // out0, out1
    const bool gelu = AUX && p.epilogue == LZ_EPI_GELU, dgelu = AUX && p.epilogue == LZ_EPI_DGELU;
    const bool swiglu = AUX && p.epilogue == LZ_EPI_SWIGLU;
    const bool dswiglu = AUX && p.epilogue == LZ_EPI_DSWIGLU;
    constexpr int kChunks = C::kTileN / kEpiCols / (kEpiWarps / 4);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = next_tile(false); tile < total; tile = next_tile(false)) {
      const TileInfo t = decode_tile<CG, NS>(p, s_pref, s_off, s_perm, total0, tile);
      const int row0 = (p.mode == 0 ? s_off[t.g] : t.g * p.c_grp_rows + p.c_row_off) +
                       t.mb * C::kTileM + cta * BM + quad * 32;
      const int col0 = t.nb * C::kTileN + half * (C::kTileN / (kEpiWarps / 4));
      if (swiglu || dswiglu) {
        swiglu_epilogue(p, swiglu, t, row0, half, lane, tmem_base + ((uint32_t)(quad * 32) << 16) +
                        acc * kAccCols, &tfull_bar[acc], acc_phase, &tempty_bar[acc], wbuf,
                        &map_c, CG);
        if (++acc == C::kNAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      // One instantiation per epilogue kind, so each has its own register allocation (the
      // dGELU aux prefetch registers are not live in the GELU path and vice versa).
      auto plain_tile = [&](auto kind) {
        constexpr int K = decltype(kind)::value;   // 0 store, 1 GELU, 2 dGELU
        // GELU / dGELU aux = gelu'(h) in the private blocked layout (aux_block): lane l
        // of the warp owning rows row0..row0+31 touches 16 B per instruction at
        // consecutive addresses -> 512 B coalesced accesses, no smem staging, no TMA
        const uint4* aux_rd = nullptr;
        uint4 hnext[4];
        if constexpr (K == 2) {
          aux_rd = aux_block(p, p.N, row0, col0) + lane;
#pragma unroll
          for (int q = 0; q < 4; ++q) hnext[q] = ld_nc_v4(aux_rd + q * 32);
        }
        // scatter epilogue: this lane's output row goes straight back (NVLink store) to
        // the rank that sent it -- the combine / dispatch-backward then read locally
        uint4* sc_dst = nullptr;
        const CUtensorMap* smap = &map_c;   // TMA store target and row of this warp's chunk
        int srow = row0;
        bool scatter = false;               // per-row direct stores (non-contiguous chunk)
        if constexpr (K == 0) {
          if (p.ret_map) {
            const long long code = __ldg(p.ret_map + row0 + lane);
            const long long cf = __shfl_sync(0xffffffffu, code, 0);
            const long long cl = __shfl_sync(0xffffffffu, code, 31);
            if (cf >= 0 && cl - cf == 31 && (cf >> 32) == (cl >> 32) && (cf >> 32) < rmaps.n) {
              smap = &rmaps.m[cf >> 32];
              srow = (int)(cf & 0xffffffffll);
            } else {
              scatter = true;
              if (code >= 0)
                sc_dst = reinterpret_cast<uint4*>(p.ret_peers[code >> 32]) +
                         (code & 0xffffffffll) * (p.N >> 3) + (col0 >> 3);
            }
          }
        }
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * kAccCols +
                               half * (C::kTileN / (kEpiWarps / 4));
#pragma unroll 1
        for (int c = 0; c < kChunks; ++c) {
          const int b = c & 1;
          uint32_t v[32];
          if (t.nk > 0) {
            tmem_ld32(taddr + c * kEpiCols, v);
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = 0u;
          }
          if (c == kChunks - 1) {
            // accumulator fully read: hand TMEM back to the MMA issuer early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) tmem_release(&tempty_bar[acc], CG);
          }
          float f[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) f[q] = __uint_as_float(v[q]);
          if constexpr (K == 2) {
            // dA * gelu'(h) (aux loaded during the previous chunk)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float h[8];
              bf16x8_to_f32(hnext[q], h);
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                const float2 m = mul2(make_float2(f[8 * q + i], f[8 * q + i + 1]),
                                      make_float2(h[i], h[i + 1]));
                f[8 * q + i] = m.x;
                f[8 * q + i + 1] = m.y;
              }
            }
            if (c + 1 < kChunks) {
#pragma unroll
              for (int q = 0; q < 4; ++q) hnext[q] = ld_nc_v4(aux_rd + (c + 1) * 128 + q * 32);
            }
          }
          if (scatter) {
            if (sc_dst) {
#pragma unroll
              for (int q = 0; q < 4; ++q) st_v4(sc_dst + c * 4 + q, f32_to_bf16x8(f + 8 * q));
            }
            continue;
          }
          // GELU: y and gelu'(y) in registers first; the aux stores are issued only AFTER
          // this chunk's smem staging + proxy fence + TMA store, so the fence (which orders
          // this thread's earlier generic-proxy writes) never waits for them
          uint4 auxv[4];
          if constexpr (K == 1) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float dg[8];
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                float2 y2, d2;
                gelu_and_grad2(make_float2(f[8 * q + i], f[8 * q + i + 1]), y2, d2);
                f[8 * q + i] = y2.x;
                f[8 * q + i + 1] = y2.y;
                dg[i] = d2.x;
                dg[i + 1] = d2.y;
              }
              auxv[q] = f32_to_bf16x8(dg);
            }
          }
          // the store that used buffer b (chunk c-2) must have finished reading smem
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(out_s + b * kEpiBuf + stg_off(lane, q), f32_to_bf16x8(f + 8 * q));
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(smap, wbuf + b * kEpiBuf, col0 + c * kEpiCols, srow);
            bulk_commit();
          }
          if constexpr (K == 1) {
            uint4* aux_wr = aux_block(p, p.N, row0, col0 + c * kEpiCols) + lane;
#pragma unroll
            for (int q = 0; q < 4; ++q) st_v4(aux_wr + q * 32, auxv[q]);
          }
        }
      };
      if (gelu) plain_tile(std::integral_constant<int, 1>{});
      else if (dgelu) plain_tile(std::integral_constant<int, 2>{});
      else plain_tile(std::integral_constant<int, 0>{});
      if (++acc == C::kNAcc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  if (CG == 1) __syncthreads();
  else cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(kTmemCols));
  }
}

}  // namespace gemm
}  // namespace lz

// ------------------------------------------------------------------------ host
using namespace lz::gemm;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 2D bf16 tensor map over a row-major [outer, inner] matrix.
static bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                     uint32_t box_inner, uint32_t box_outer,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn enc = get_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int g_cta_group = 2;  // default: CTA-pair kernel

// Dynamic tile scheduler counters (Params::tile_ctr): a rolling pool of counter pairs, one
// per launch, each reset to zero by the last unit of its launch (so a slot is reusable,
// also by every replay of a captured graph).  LZ_GEMM_DYNAMIC=0 keeps the static schedule.
constexpr int kCtrSlots = 1024;
__device__ int g_tile_ctr[kCtrSlots][2];
// Policy: LZ_GEMM_DYNAMIC=1 always dynamic, 2 = dynamic for the weight-gradient GEMMs and
// the reduced-grid row GEMMs next to NCCL only, unset / 0 = the static snake schedule.
// Measured (profiles/r02_gemm_dynamic_ab.log): launched alone, the weight-gradient GEMMs are
// 13-20 % faster dynamic and the short-K row GEMMs 6-8 % slower; inside the whole step
// (N = 1 and N = 4, interleaved runs) neither policy beats the static schedule beyond
// run-to-run noise, so the static one stays the default.
static int* tile_counter(int mode, int num_sms) {
  static const int pol = [] {
    const char* e = getenv("LZ_GEMM_DYNAMIC");
    return e ? atoi(e) : 0;
  }();
  const bool on = pol == 1 || (pol == 2 && (mode == 1 || num_sms > 0));
  if (!on) return nullptr;
  static int* base = nullptr;
  static unsigned next = 0;
  if (!base) {
    void* ptr = nullptr;
    if (cudaGetSymbolAddress(&ptr, g_tile_ctr) != cudaSuccess) return nullptr;
    base = (int*)ptr;
  }
  return base + 2 * (next++ % kCtrSlots);
}
// L2 budget of the re-read operand chunk (Params::l2_chunk_bytes); LZ_GEMM_L2_CHUNK_MB
// overrides it for A/B runs (0 = no chunking: plain inner-fastest raster)
static long long g_l2_chunk_bytes = [] {
  const char* e = getenv("LZ_GEMM_L2_CHUNK_MB");
  const long long mb = e ? atoll(e) : 40;
  return mb > 0 ? mb << 20 : (1ll << 62);
}();

LZ_DEFINE_CTL_SETTER(lz_gemm_set_control_internal)

extern "C" int lz_gemm_set_cta_group(int cg) {
  if (cg == 1 || cg == 2) g_cta_group = cg;
  return g_cta_group;
}
extern "C" int lz_gemm_row_align(void) { return BM * g_cta_group; }

template <int A_MN, int B_MN, int CG, bool AUX, int NS = 1>
static lz_status launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                        const CUtensorMap& mx, const Params& p, const RetMaps& rm, int grid,
                        cudaStream_t s) {
  auto kern = grouped_gemm_kernel<A_MN, B_MN, CG, AUX, NS>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg<CG, AUX, NS>::kSmemBytes) != cudaSuccess)
      return lzh::check_launch();
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg<CG, AUX, NS>::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // pdl_prologue
  attr[1].val.programmaticStreamSerializationAllowed = lzh::pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mx, p, rm) != cudaSuccess)
    return lzh::check_launch();
  return lzh::check_launch();
}

// 256 x 512 tiles (Cfg NS = 2) for the store-epilogue GEMMs with a long main loop: the
// weight gradients (K = an expert's rows) and row GEMMs with K >= 2048 (the one-accumulator
// epilogue is then a few % of a tile); N % 512 == 0.  LZ_GEMM_WIDE=0 keeps 256 x 256, =2
// only the weight gradients.
static bool wide_tiles(int mode, int N, int K) {
  static const int on = [] {
    const char* e = getenv("LZ_GEMM_WIDE");
    return e ? atoi(e) : 1;
  }();
  if (on == 0 || N % (2 * BN)) return false;
  return mode == 1 || (on == 1 && K >= 2048);
}

template <int A_MN, int B_MN, bool AUX>
static lz_status launch_cg(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                           const CUtensorMap& mx, const Params& p, const RetMaps& rm, long tiles,
                           int sms, cudaStream_t s) {
  if (g_cta_group == 2) {
    long units = tiles < sms / 2 ? tiles : sms / 2;
    if (units < 1) units = 1;
    if constexpr (!AUX) {
      if (wide_tiles(p.mode, p.N, p.K)) {
        const long t2 = tiles / 2;   // 256 x 512 tiles
        long u2 = t2 < sms / 2 ? t2 : sms / 2;
        if (u2 < 1) u2 = 1;
        return launch<A_MN, B_MN, 2, AUX, 2>(ma, mb, mc, mx, p, rm, (int)(2 * u2), s);
      }
    }
    return launch<A_MN, B_MN, 2, AUX>(ma, mb, mc, mx, p, rm, (int)(2 * units), s);
  }
  long grid = tiles < sms ? tiles : sms;
  if (grid < 1) grid = 1;
  return launch<A_MN, B_MN, 1, AUX>(ma, mb, mc, mx, p, rm, (int)grid, s);
}
template <int A_MN, int B_MN>
static lz_status launch_cg(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                           const CUtensorMap& mx, const Params& p, const RetMaps& rm, long tiles,
                           int sms, cudaStream_t s) {
  return p.epilogue == LZ_EPI_STORE
             ? launch_cg<A_MN, B_MN, false>(ma, mb, mc, mx, p, rm, tiles, sms, s)
             : launch_cg<A_MN, B_MN, true>(ma, mb, mc, mx, p, rm, tiles, sms, s);
}

static lz_status grouped_gemm_impl(int mode, const void* A, const void* B, void* C, void* aux,
                                   int G, const int32_t* off, int rows_total, int M, int N,
                                   int K, int b_major, int epilogue, int num_sms,
                                   int c_group_rows, int c_row_offset, void* stream,
                                   const long long* ret_map, const unsigned long long* ret_peers,
                                   const RetMaps& rm, const int32_t* self_rows = nullptr,
                                   const int* flags = nullptr, int n_flags = 0,
                                   const int* epoch = nullptr);

extern "C" lz_status lz_grouped_gemm_arrival(const void* A, const void* B, void* C, void* aux,
                                             int G, const int32_t* off, int rows_total, int N,
                                             int K, int b_major, int epilogue, int num_sms,
                                             const int32_t* self_rows, const int* flags,
                                             int n_flags, const int* epoch, void* stream) {
  if (!self_rows || !flags || !epoch || n_flags < 1) return LZ_ERR_ARG;
  static const RetMaps none{};
  return grouped_gemm_impl(0, A, B, C, aux, G, off, rows_total, 0, N, K, b_major, epilogue,
                           num_sms, 0, 0, stream, nullptr, nullptr, none, self_rows, flags,
                           n_flags, epoch);
}

extern "C" lz_status lz_grouped_gemm(int mode, const void* A, const void* B, void* C, void* aux,
                                     int G, const int32_t* off, int rows_total, int M, int N,
                                     int K, int b_major, int epilogue, int num_sms,
                                     int c_group_rows, int c_row_offset, void* stream) {
  static const RetMaps none{};
  return grouped_gemm_impl(mode, A, B, C, aux, G, off, rows_total, M, N, K, b_major, epilogue,
                           num_sms, c_group_rows, c_row_offset, stream, nullptr, nullptr, none);
}

extern "C" lz_status lz_grouped_gemm_scatter(const void* A, const void* B, void* C, int G,
                                             const int32_t* off, int rows_total, int N, int K,
                                             int b_major, int num_sms,
                                             const long long* ret_map,
                                             const unsigned long long* ret_peers,
                                             const unsigned long long* ret_peers_host,
                                             int n_peers, int ret_rows, void* stream) {
  if (!ret_map || !ret_peers || n_peers < 0 || ret_rows < 0 || (n_peers > 0 && !ret_peers_host))
    return LZ_ERR_ARG;
  RetMaps rm{};
  rm.n = n_peers <= kMaxRetPeers ? n_peers : 0;   // more ranks: per-row stores only
  for (int r = 0; r < rm.n; ++r)
    if (!make_map(&rm.m[r], (void*)ret_peers_host[r], N, ret_rows > 0 ? ret_rows : 1, kEpiCols,
                  32, CU_TENSOR_MAP_SWIZZLE_64B))
      return LZ_ERR_CUDA;
  return grouped_gemm_impl(0, A, B, C, nullptr, G, off, rows_total, 0, N, K, b_major,
                           LZ_EPI_STORE, num_sms, 0, 0, stream, ret_map, ret_peers, rm);
}

static lz_status grouped_gemm_impl(int mode, const void* A, const void* B, void* C, void* aux,
                                   int G, const int32_t* off, int rows_total, int M, int N,
                                   int K, int b_major, int epilogue, int num_sms,
                                   int c_group_rows, int c_row_offset, void* stream,
                                   const long long* ret_map, const unsigned long long* ret_peers,
                                   const RetMaps& rm, const int32_t* self_rows, const int* flags,
                                   int n_flags, const int* epoch) {
  if (G < 1 || !A || !B || !C || !off || rows_total < 0) return LZ_ERR_ARG;
  if (G > kMaxGroups) return LZ_ERR_UNSUPPORTED;
  if (epilogue < LZ_EPI_STORE || epilogue > LZ_EPI_DSWIGLU) return LZ_ERR_ARG;
  if ((epilogue != LZ_EPI_STORE) && (mode != 0 || !aux)) return LZ_ERR_ARG;
  if (N <= 0 || N % BN) return LZ_ERR_UNSUPPORTED;
  const int tile_m = BM * g_cta_group;
  CUtensorMap ma, mb, mc, mx;
  Params p{};
  p.mode = mode;
  p.G = G;
  p.M = M;
  p.N = N;
  p.K = K;
  p.off = off;
  p.epilogue = epilogue;
  p.c_grp_rows = c_group_rows > 0 ? c_group_rows : M;
  p.c_row_off = c_row_offset;
  p.C = (__nv_bfloat16*)C;
  p.aux = (__nv_bfloat16*)aux;
  p.ret_map = ret_map;
  p.ret_peers = ret_peers;
  p.self_rows = self_rows;
  p.flags = flags;
  p.n_flags = n_flags;
  p.epoch = epoch;
  p.l2_chunk_bytes = g_l2_chunk_bytes;
  p.tile_ctr = tile_counter(mode, num_sms);
  cudaStream_t s = (cudaStream_t)stream;
  int sms = num_sms > 0 ? num_sms : lzh::num_sms();
  if (sms < 2) sms = 2;
  if (rows_total == 0 && mode == 0) return LZ_OK;
  const CUtensorMapSwizzle sw64 = CU_TENSOR_MAP_SWIZZLE_64B;
  const int brows = BN / g_cta_group;
  if (mode == 0) {
    if (K <= 0 || K % BK) return LZ_ERR_UNSUPPORTED;
    if (!make_map(&ma, A, K, rows_total, BK, BM)) return LZ_ERR_CUDA;
    if (b_major == LZ_K_MAJOR) {
      if (!make_map(&mb, B, K, (uint64_t)G * N, BK, brows)) return LZ_ERR_CUDA;
    } else {
      if (!make_map(&mb, B, N, (uint64_t)G * K, 64, BK)) return LZ_ERR_CUDA;
    }
    // output / aux widths: SWIGLU writes C[rows, N/2] and H[rows, N]; DSWIGLU reads and
    // writes the interleaved [rows, 2N]
    const uint64_t c_w = epilogue == LZ_EPI_SWIGLU ? N / 2 : (epilogue == LZ_EPI_DSWIGLU ? 2 * N : N);
    const uint64_t x_w = epilogue == LZ_EPI_DSWIGLU ? 2 * N : N;
    if (!make_map(&mc, C, c_w, rows_total, kEpiCols, 32, sw64)) return LZ_ERR_CUDA;
    if (!make_map(&mx, aux ? aux : C, x_w, rows_total, kEpiCols, 32, sw64)) return LZ_ERR_CUDA;
    // upper bound of tiles; the kernel reads the exact count from the device offsets
    long tiles = (long)(rows_total / tile_m) * (N / BN);
    return b_major == LZ_K_MAJOR ? launch_cg<0, 0>(ma, mb, mc, mx, p, rm, tiles, sms, s)
                                 : launch_cg<0, 1>(ma, mb, mc, mx, p, rm, tiles, sms, s);
  } else if (mode == 1) {
    if (M <= 0 || M % tile_m) return LZ_ERR_UNSUPPORTED;
    if (c_group_rows != 0 && (c_group_rows < M || c_row_offset < 0 ||
                              c_row_offset + M > c_group_rows))
      return LZ_ERR_ARG;
    const uint64_t rows = rows_total > 0 ? rows_total : 1;
    if (!make_map(&ma, A, M, rows, 64, BK)) return LZ_ERR_CUDA;
    if (!make_map(&mb, B, N, rows, 64, BK)) return LZ_ERR_CUDA;
    const uint64_t c_rows = (uint64_t)(G - 1) * p.c_grp_rows + c_row_offset + M;
    if (!make_map(&mc, C, N, c_rows, kEpiCols, 32, sw64)) return LZ_ERR_CUDA;
    long tiles = (long)G * (M / tile_m) * (N / BN);
    return launch_cg<1, 1>(ma, mb, mc, mc, p, rm, tiles, sms, s);
  }
  return LZ_ERR_ARG;
}
