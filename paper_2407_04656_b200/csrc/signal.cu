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

}  // namespace lz

using namespace lz;

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
