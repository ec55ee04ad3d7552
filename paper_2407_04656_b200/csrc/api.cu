// api.cu -- library-level entry points of liblz.so (status strings, version).
#include "common.cuh"

extern "C" const char* lz_status_string(int status) {
  switch (status) {
    case LZ_OK: return "ok";
    case LZ_ERR_ARG: return "invalid argument";
    case LZ_ERR_UNROUTABLE: return "tokens routed to an expert without replicas";
    case LZ_ERR_CUDA: return "CUDA error";
    case LZ_ERR_WORKSPACE: return "workspace too small";
    case LZ_ERR_UNSUPPORTED: return "shape outside compiled limits";
    default: return "unknown status";
  }
}

extern "C" int lz_version(void) { return 100; }  // 0.1.0

extern "C" int lz_last_cuda_error(void) { return lzh::last_cuda_error(); }

extern "C" lz_status lz_gemm_set_control_internal(lz_ctl* c);
extern "C" lz_status lz_signal_set_control_internal(lz_ctl* c);

// Every module that waits on peers or on its own pipeline keeps its own copy of the
// control-block pointer (lz.h lz_ctl).
extern "C" lz_status lz_set_control(lz_ctl* ctl) {
  lz_status st = lz_gemm_set_control_internal(ctl);
  if (st != LZ_OK) return st;
  return lz_signal_set_control_internal(ctl);
}
