// pipeoptim_gemm_stub.cpp — linked instead of pipeoptim_gemm.cu when no CUTLASS
// header tree is found at build time (build.py). The optimizer, stage-op, LSTM
// and transport kernels never need CUTLASS; only the fp32 tensor-core stage
// GEMM does, and without it the stage math runs on cuBLAS (stages._tc_ok).
#include <stdint.h>

#include "pipeoptim.h"

extern "C" {

int po_gemm_f32x3_available(void) { return 0; }

int po_set_gemm_tile(int32_t tile_n) { return (tile_n == 64 || tile_n == 128) ? 0 : PO_EINVAL; }

int po_get_gemm_tile(void) { return 64; }

int po_gemm_f32x3(int32_t, int32_t, const float*, int64_t, int64_t, const float*, int64_t, int64_t, float*, int64_t,
                  int64_t, int64_t, int64_t, void*, int64_t, void*) {
  return PO_ENOSYS;
}

}  // extern "C"
