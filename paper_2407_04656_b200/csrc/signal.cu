// signal.cu -- arrival flags of the multi-GPU exchange (no reference counterpart: the
// reference has no data plane).
//
// After a rank's dispatch kernel has stored its rows into the owners' symmetric receive
// buffers, lz_signal_peers publishes this step's epoch into every owner's flag slot for
// this sender (system-scope release).  The owners' arrival-ordered GEMM
// (lz_grouped_gemm_arrival) runs the tiles made of their own rows first and acquires the
// flags only before the first tile that holds rows from other ranks -- the dispatch
// all-to-all overlaps the first GEMM instead of sitting behind a full barrier.
#include "common.cuh"

namespace lz {

__global__ void epoch_bump_kernel(int* epoch) { *epoch += 1; }

__global__ void signal_peers_kernel(const unsigned long long* __restrict__ flag_peers, int n,
                                    int my_rank, const int* __restrict__ epoch) {
  __threadfence_system();   // the dispatch kernel's remote stores before the flags
  const int lane = threadIdx.x;
  if (lane < n) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(epoch) : "memory");
    int* f = reinterpret_cast<int*>(flag_peers[lane]) + my_rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  }
}

// One warp per participating rank (one warp per launch across GPUs; every co-hosted
// rank in ONE block when several ranks share a GPU, so the waiting warps are co-resident
// by construction): lane j publishes the new count into rank j's barrier row, then lane i
// waits for rank i's count in ours.  Bounded by the control block (peer_wait_give_up).
__global__ void peer_barrier_kernel(const unsigned long long* __restrict__ flag_peers, int n,
                                    const int* __restrict__ ranks, int my_rank0,
                                    const unsigned long long* __restrict__ counter_ptrs,
                                    int* __restrict__ counter0,
                                    const unsigned long long* __restrict__ own_flag_ptrs,
                                    const int* __restrict__ own_flags0) {
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const int my_rank = ranks ? ranks[w] : my_rank0;
  int* counter = counter_ptrs ? reinterpret_cast<int*>(counter_ptrs[w]) : counter0;
  const int* own_flags = own_flag_ptrs ? reinterpret_cast<const int*>(own_flag_ptrs[w])
                                       : own_flags0;
  int v = 0;
  if (lane == 0) {
    v = *counter + 1;
    *counter = v;   // only this kernel touches the counter, stream-ordered
  }
  v = __shfl_sync(0xffffffffu, v, 0);
  __threadfence_system();   // every earlier write of this rank (incl. remote) before the flag
  if (lane < n) {
    int* f = reinterpret_cast<int*>(flag_peers[lane]) + my_rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
    long long deadline = 0;
    for (;;) {
      int got;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(got) : "l"(own_flags + lane)
                   : "memory");
      if (got - v >= 0) break;
      if (peer_wait_give_up(deadline)) break;
    }
  }
  __syncwarp();
}

}  // namespace lz

using namespace lz;

LZ_DEFINE_CTL_SETTER(lz_signal_set_control_internal)

extern "C" lz_status lz_peer_barrier(const unsigned long long* flag_peers, int n, int my_rank,
                                     int* counter, const int* own_flags, void* stream) {
  if (!flag_peers || !counter || !own_flags || n < 1 || n > 32 || my_rank < 0 || my_rank >= n)
    return LZ_ERR_ARG;
  peer_barrier_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(flag_peers, n, nullptr, my_rank,
                                                          nullptr, counter, nullptr, own_flags);
  return lzh::check_launch();
}

extern "C" lz_status lz_peer_barrier_colocated(const unsigned long long* flag_peers, int n,
                                               const int* ranks, int n_local,
                                               const unsigned long long* counter_ptrs,
                                               const unsigned long long* own_flag_ptrs,
                                               void* stream) {
  if (!flag_peers || !ranks || !counter_ptrs || !own_flag_ptrs || n < 1 || n > 32 ||
      n_local < 1 || n_local > 32)
    return LZ_ERR_ARG;
  peer_barrier_kernel<<<1, 32 * n_local, 0, (cudaStream_t)stream>>>(
      flag_peers, n, ranks, 0, counter_ptrs, nullptr, own_flag_ptrs, nullptr);
  return lzh::check_launch();
}

extern "C" lz_status lz_epoch_bump(int* epoch, void* stream) {
  if (!epoch) return LZ_ERR_ARG;
  epoch_bump_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(epoch);
  return lzh::check_launch();
}

extern "C" lz_status lz_signal_peers(const unsigned long long* flag_peers, int n, int my_rank,
                                     const int* epoch, void* stream) {
  if (!flag_peers || !epoch || n < 1 || n > 32 || my_rank < 0 || my_rank >= n) return LZ_ERR_ARG;
  signal_peers_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(flag_peers, n, my_rank, epoch);
  return lzh::check_launch();
}
