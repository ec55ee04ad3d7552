// common.cuh -- shared helpers for liblz (sm_100a only).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "../../include/lz.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "liblz targets sm_100a only"
#endif

namespace lz {

constexpr int kWarp = 32;

__device__ __forceinline__ unsigned lane_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// 16-byte streaming loads/stores (read-once activations: do not allocate in L1)
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void bf16x8_to_f32(uint4 v, float* f) {
  const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(u[i] << 16);
    f[2 * i + 1] = __uint_as_float(u[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // .x = a (low), .y = b (high)
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint4 f32_to_bf16x8(const float* f) {
  uint4 v;
  v.x = pack_bf16x2(f[0], f[1]);
  v.y = pack_bf16x2(f[2], f[3]);
  v.z = pack_bf16x2(f[4], f[5]);
  v.w = pack_bf16x2(f[6], f[7]);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- watchdog / abort control block (lz.h lz_ctl) ----------------------------------
// One device-global pointer per translation unit (the .cu files are separate modules);
// LZ_DEFINE_CTL_SETTER gives each module that waits on peers its setter, lz_set_control
// (api.cu) calls them all.
static __device__ lz_ctl* g_ctl = nullptr;

__device__ __forceinline__ long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (long long)t;
}
__device__ __forceinline__ int ld_sys_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_sys_s32(int* p, int v) {
  asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ long long ctl_timeout_ns() {
  const lz_ctl* c = g_ctl;
  const long long t = c ? c->timeout_ns : 0;
  return t > 0 ? t : 10000000000ll;
}
// Poll step of a bounded cross-rank wait that has not succeeded yet: sleeps briefly, and
// returns true (after recording the cause) when the wait must give up.
__device__ __forceinline__ bool peer_wait_give_up(long long& deadline) {
  const long long now = globaltimer_ns();
  if (deadline == 0) deadline = now + ctl_timeout_ns();
  lz_ctl* c = g_ctl;
  if (c && ld_sys_s32(&c->abort)) {
    st_sys_s32(&c->aborted, 1);
    return true;
  }
  if (now > deadline) {
    if (c) st_sys_s32(&c->timeout, 1);
    return true;
  }
  // a wait that already gave up elsewhere in this step: do not stack another full timeout
  if (c && (ld_sys_s32(&c->timeout) | ld_sys_s32(&c->aborted))) return true;
  __nanosleep(256);
  return false;
}

// ---- programmatic dependent launch (PDL) ------------------------------------------------
// Kernels of the step's chain are launched with programmatic stream serialisation
// (lzh::launch): each lets its dependents launch as soon as all of its blocks are running
// and waits for its own predecessor's completion (and memory) before touching its
// outputs, so a kernel's launch and prologue overlap the previous kernel's tail.
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// The two halves, for kernels with a prologue that touches no global memory a predecessor
// may write (barrier init, TMEM allocation, staging of weights no kernel of the chain
// writes): launch_dependents first, the prologue, then wait before any other global
// access -- the prologue overlaps the predecessor's tail.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Softmax / top-k (/ renorm) backward of one token (the gate backward):
// with the k routed ids' probabilities ps and upstream weight gradients g (= dw),
//   renorm: g_s <- (g_s - sum_s' g_s' ps_s' / S) / S,  S = sum_s ps_s
//   dot = sum_s g_s ps_s,   dlogits_e = -p_e dot + sum_s [e == id_s] ps_s g_s.
// Returns dot and turns g into the coefficients c_s = ps_s g_s.  Explicit roundings, so
// every kernel that evaluates it (lz_gate_bwd, lz_dispatch_bwd) gets identical bits.
__device__ __forceinline__ float gate_bwd_coefs(int k, int renorm, const float* ps, float* g) {
  float S = 0.f;
#pragma unroll
  for (int s = 0; s < LZ_MAX_TOPK; ++s)
    if (s < k) S = __fadd_rn(S, ps[s]);
  if (renorm) {
    float sdw = 0.f;
#pragma unroll
    for (int s = 0; s < LZ_MAX_TOPK; ++s)
      if (s < k) sdw = __fmaf_rn(g[s], __fdiv_rn(ps[s], S), sdw);
#pragma unroll
    for (int s = 0; s < LZ_MAX_TOPK; ++s)
      if (s < k) g[s] = __fdiv_rn(__fsub_rn(g[s], sdw), S);
  }
  float dot = 0.f;
#pragma unroll
  for (int s = 0; s < LZ_MAX_TOPK; ++s)
    if (s < k) dot = __fmaf_rn(g[s], ps[s], dot);
#pragma unroll
  for (int s = 0; s < LZ_MAX_TOPK; ++s) g[s] = s < k ? __fmul_rn(ps[s], g[s]) : 0.f;
  return dot;
}
// dlogits_e of expert e from gate_bwd_coefs' results (ids of unused slots are -1)
__device__ __forceinline__ float gate_bwd_dl(float p_e, int e, float dot, const int* ids,
                                             const float* c) {
  float v = __fmul_rn(-p_e, dot);
#pragma unroll
  for (int s = 0; s < LZ_MAX_TOPK; ++s)
    if (ids[s] == e) v = __fadd_rn(v, c[s]);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace lz

// host-side helpers shared by the api translation units
namespace lzh {
inline int& last_cuda_error() {
  static thread_local int e = 0;
  return e;
}
inline lz_status check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    last_cuda_error() = (int)e;
    return LZ_ERR_CUDA;
  }
  return LZ_OK;
}
inline bool pdl_enabled() {
  static const int on = [] {
    const char* e = getenv("LZ_PDL");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}
// cudaLaunchKernelEx with programmatic stream serialisation (see pdl_prologue) and an
// optional cluster size; every kernel launched this way calls pdl_prologue() first.
template <typename... KArgs, typename... Args>
inline lz_status launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                        cudaStream_t s, int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[na].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  ++na;
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  return check_launch();
}
inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}
}  // namespace lzh

#define LZ_DEFINE_CTL_SETTER(name)                                          \
  extern "C" lz_status name(lz_ctl* c) {                                    \
    if (cudaMemcpyToSymbol(lz::g_ctl, &c, sizeof(c)) == cudaSuccess)        \
      return LZ_OK;                                                         \
    lzh::check_launch();                                                    \
    return LZ_ERR_CUDA;                                                     \
  }
