// reliability.cu -- exact recovery probability under k uniform node failures
// (reference reliability.py:68-96 recovery_probability_exact).
//
// The reference enumerates every alive set of size N - k in Python (capped at 10^6
// subsets).  Here every failed set F of size k (same count, C(N, k) = C(N, N - k)) is a
// 64-bit node mask; thread ranges of consecutive colex ranks are unranked with the
// combinatorial number system and advanced with Gosper's hack.  The state is
// recoverable iff every expert keeps a surviving holder: (holders_e & ~F) != 0 for all
// e.  The count of recoverable sets is exact (integer), so Fraction(good, total) is
// bit-identical to the reference's.
#include "common.cuh"

namespace lz {

__constant__ unsigned long long c_binom[65][65];

__device__ __forceinline__ unsigned long long unrank_colex(unsigned long long rank, int k, int n) {
  // largest c with C(c, i) <= rank, for i = k .. 1 (combinatorial number system)
  unsigned long long mask = 0;
  int c = n - 1;
  for (int i = k; i >= 1; --i) {
    while (c >= i && c_binom[c][i] > rank) --c;
    if (c < i - 1) c = i - 1;
    if (c_binom[c][i] <= rank) rank -= c_binom[c][i];
    mask |= 1ull << c;
    --c;
  }
  return mask;
}

__device__ __forceinline__ unsigned long long gosper_next(unsigned long long x) {
  // next larger integer with the same popcount (colex successor of the subset)
  const unsigned long long u = x & (~x + 1ull);
  const unsigned long long v = x + u;
  return v + ((v ^ x) >> (__ffsll((long long)u) + 1));
}

__global__ void __launch_bounds__(256) recovery_count_kernel(
    const unsigned long long* __restrict__ holders, int E, int n, int k,
    unsigned long long total, unsigned long long per_thread, unsigned long long* __restrict__ good) {
  __shared__ unsigned long long s_h[1024];
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_h[e] = holders[e];
  __syncthreads();
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long r0 = tid * per_thread;
  unsigned long long cnt = 0;
  if (r0 < total) {
    const unsigned long long r1 = r0 + per_thread < total ? r0 + per_thread : total;
    unsigned long long f = k == 0 ? 0ull : unrank_colex(r0, k, n);
    for (unsigned long long r = r0; r < r1; ++r) {
      bool ok = true;
      for (int e = 0; e < E; ++e)
        if ((s_h[e] & ~f) == 0ull) {
          ok = false;
          break;
        }
      cnt += ok;
      if (k > 0 && r + 1 < r1) f = gosper_next(f);
    }
  }
  // warp sum, one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(good, cnt);
}

}  // namespace lz

using namespace lz;

extern "C" lz_status lz_recovery_count(const unsigned long long* holders, int E, int n_nodes,
                                       int k_failed, unsigned long long* good, void* stream) {
  if (E < 1 || E > 1024 || n_nodes < 1 || n_nodes > 63 || k_failed < 0 || k_failed > n_nodes ||
      !holders || !good)
    return LZ_ERR_ARG;
  static bool table = false;
  static unsigned long long binom[65][65];
  if (!table) {
    for (int a = 0; a <= 64; ++a)
      for (int b = 0; b <= 64; ++b)
        binom[a][b] = b == 0 ? 1ull : (a == 0 ? 0ull : binom[a - 1][b - 1] + binom[a - 1][b]);
    if (cudaMemcpyToSymbol(c_binom, binom, sizeof(binom)) != cudaSuccess) return lzh::check_launch();
    table = true;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(good, 0, sizeof(unsigned long long), s) != cudaSuccess)
    return lzh::check_launch();
  const unsigned long long total = binom[n_nodes][k_failed];
  // ~ 8 waves of 256-thread blocks over the SMs, at least 64 sets per thread
  const unsigned long long threads = (unsigned long long)lzh::num_sms() * 2048ull * 8ull;
  unsigned long long per = (total + threads - 1) / threads;
  if (per < 64) per = 64;
  const unsigned long long nthreads = (total + per - 1) / per;
  const unsigned long long blocks = (nthreads + 255) / 256;
  if (blocks > 0x7fffffffull) return LZ_ERR_UNSUPPORTED;
  recovery_count_kernel<<<(unsigned)blocks, 256, 0, s>>>(holders, E, n_nodes, k_failed, total, per,
                                                         good);
  return lzh::check_launch();
}
