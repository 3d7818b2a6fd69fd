// pipeoptim_gemm.cu — FP32-accurate stage GEMMs on the tcgen05 tensor cores.
//
// The config-1 stage GEMMs are fp32 (the parity contract keeps TF32 off), so
// cuBLAS runs them on the CUDA cores (SIMT SGEMM, 74 TFLOP/s peak, 13-35
// TFLOP/s achieved at these shapes). This TU instantiates CUTLASS's SM100
// "fast FP32" mainloop: each fp32 operand is split into three bf16 pieces in
// shared memory and the products are accumulated in fp32 in TMEM by
// tcgen05.mma (UMMA) — fp32-level accuracy at tensor-core throughput. It is
// used as a batched GEMM so the caller can run the small-M, long-K stage
// shapes split-K (batch = K slice) and reduce the partials in its own fused
// epilogue (po_splitk_bias_act / po_act_bwd_bias).
//
//   D[l] (M x N, row-major) = A[l] (M x K) @ B[l] (K x N)
//   A: row-major with leading dimension lda (K-major), batch stride sa
//   B: row-major K x N with leading dimension ldb (N-major), batch stride sb
//   D: row-major, leading dimension N, batch stride M*N
#include <cuda_runtime.h>
#include <stdint.h>

// The kernels are launched with programmatic dependent launch (PDL); with this
// set, CUTLASS's producer waits on the preceding grid (griddepcontrol.wait)
// before its first operand load — without it the wait compiles to nothing.
#define CUTLASS_ENABLE_GDC_FOR_SM100 1

#include "cute/tensor.hpp"
#include "cutlass/cutlass.h"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"
#include "pipeoptim.h"

namespace {

using namespace cute;

using ElementAcc = float;
using LayoutD = cutlass::layout::RowMajor;
constexpr int kAlign = 4;  // 16-byte TMA alignment in floats

#ifndef PO_FASTF32_TILE_N  // the default tile width (po_set_gemm_tile selects 64 or 128 at run time)
#define PO_FASTF32_TILE_N 64
#endif
#ifndef PO_FASTF32_TILE_K
#define PO_FASTF32_TILE_K 32
#endif
#ifndef PO_FASTF32_KMAJOR_A_SCHEDULE  // K-major A: bf16 pieces staged in shared memory (Smem) or TMEM
#define PO_FASTF32_KMAJOR_A_SCHEDULE KernelTmaWarpSpecialized1SmFastFP32SmemSm100
#endif
#ifndef PO_FASTF32_EXTRA_CARVEOUT  // bytes held back from the stage count (fewer stages, more CTAs per SM)
#define PO_FASTF32_EXTRA_CARVEOUT 0
#endif
using ClusterShape = Shape<_1, _1, _1>;

// One epilogue per tile shape; one mainloop per (tile width, operand-major
// pair). Two tile widths: 128 x 64 (more CTAs: the lowest latency for a
// stage alone on its GPU) and 128 x 128 (half the CTAs: less SM time per
// GEMM, the faster choice when several stages share one GPU —
// profiles/r2_gemm_tile_shared_gpu.jsonl).
template <int TN>
struct Tiles {
  using MmaTileShape = Shape<_128, Int<TN>, Int<PO_FASTF32_TILE_K>>;
  using CollectiveEpilogue = typename cutlass::epilogue::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, MmaTileShape, ClusterShape,
      cutlass::epilogue::collective::EpilogueTileAuto, ElementAcc, ElementAcc, void, LayoutD, kAlign, float,
      LayoutD, kAlign, cutlass::epilogue::collective::EpilogueScheduleAuto>::CollectiveOp;
  static constexpr int kEpiCarveout =
      static_cast<int>(sizeof(typename CollectiveEpilogue::SharedStorage)) + PO_FASTF32_EXTRA_CARVEOUT;
};

template <int TN, class LayoutA, class LayoutB, class Schedule>
struct FastF32Gemm {
  using T = Tiles<TN>;
  using Mainloop = typename cutlass::gemm::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, float, LayoutA, kAlign, float, LayoutB, kAlign,
      ElementAcc, typename T::MmaTileShape, ClusterShape,
      cutlass::gemm::collective::StageCountAutoCarveout<T::kEpiCarveout>, Schedule>::CollectiveOp;
  using Kernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Mainloop,
                                                      typename T::CollectiveEpilogue, void>;
  using Gemm = cutlass::gemm::device::GemmUniversalAdapter<Kernel>;
};

using cutlass::layout::ColumnMajor;
using cutlass::layout::RowMajor;
using SmemSched = cutlass::gemm::KernelTmaWarpSpecialized1SmFastFP32SmemSm100;
using KmajSched = cutlass::gemm::PO_FASTF32_KMAJOR_A_SCHEDULE;
template <int TN> using RowRowT = FastF32Gemm<TN, RowMajor, RowMajor, KmajSched>;     // x @ W
template <int TN> using ColRowT = FastF32Gemm<TN, ColumnMajor, RowMajor, SmemSched>;  // x^T @ dpre (M-major A)
template <int TN> using RowColT = FastF32Gemm<TN, RowMajor, ColumnMajor, KmajSched>;  // dpre @ W^T

template <class G>
int run_gemm(typename G::Gemm::GemmKernel::StrideA sa_, typename G::Gemm::GemmKernel::StrideB sb_, const float* a,
             const float* b, float* d, int64_t m, int64_t n, int64_t k, int64_t batch, void* workspace,
             int64_t workspace_bytes, cudaStream_t stream) {
  using Gemm = typename G::Gemm;
  typename Gemm::GemmKernel::StrideD stride_d =
      cute::make_stride(static_cast<int64_t>(n), cute::Int<1>{}, static_cast<int64_t>(m * n));
  cutlass::KernelHardwareInfo hw;
  hw.device_id = 0;
  cudaGetDevice(&hw.device_id);
  static int sms = 0;
  if (sms == 0) sms = cutlass::KernelHardwareInfo::query_device_multiprocessor_count(hw.device_id);
  hw.sm_count = sms;
  typename Gemm::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm,
                                {static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                                 static_cast<int>(batch)},
                                {a, sa_, b, sb_},
                                {{1.0f, 0.0f}, nullptr, stride_d, d, stride_d},
                                hw};
  Gemm gemm;
  if (gemm.can_implement(args) != cutlass::Status::kSuccess) return PO_EINVAL;
  const size_t need = Gemm::get_workspace_size(args);
  if (need > 0 && (workspace == nullptr || static_cast<size_t>(workspace_bytes) < need)) return PO_EINVAL;
  if (gemm.initialize(args, workspace, stream) != cutlass::Status::kSuccess) return PO_EINVAL;
  // programmatic dependent launch: the GEMM's CTAs are scheduled while the
  // preceding kernel drains and wait (griddepcontrol.wait) before touching
  // its operands, hiding the launch gap on the stage's critical path
  if (gemm.run(stream, nullptr, /*launch_with_pdl=*/true) != cutlass::Status::kSuccess) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PO_EINVAL : (int)e;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

// tile width of the next po_gemm_f32x3 calls (po_set_gemm_tile; process-wide)
int g_tile_n = PO_FASTF32_TILE_N;

template <int TN>
int dispatch_gemm(int32_t a_col_major, int32_t b_col_major, const float* a, int64_t lda, int64_t sa, const float* b,
                  int64_t ldb, int64_t sb, float* d, int64_t m, int64_t n, int64_t k, int64_t batch,
                  void* workspace, int64_t workspace_bytes, cudaStream_t s) {
  if (!a_col_major && !b_col_major) {  // A (m,k) at m*lda + k; B (k,n) at k*ldb + n
    if (lda < k || ldb < n) return PO_EINVAL;
    return run_gemm<RowRowT<TN>>(cute::make_stride(lda, cute::Int<1>{}, sa),
                                 cute::make_stride(cute::Int<1>{}, ldb, sb), a, b, d, m, n, k, batch, workspace,
                                 workspace_bytes, s);
  }
  if (a_col_major && !b_col_major) {  // A (m,k) at m + k*lda
    if (lda < m || ldb < n) return PO_EINVAL;
    return run_gemm<ColRowT<TN>>(cute::make_stride(cute::Int<1>{}, lda, sa),
                                 cute::make_stride(cute::Int<1>{}, ldb, sb), a, b, d, m, n, k, batch, workspace,
                                 workspace_bytes, s);
  }
  if (!a_col_major && b_col_major) {  // B (k,n) at k + n*ldb
    if (lda < k || ldb < k) return PO_EINVAL;
    return run_gemm<RowColT<TN>>(cute::make_stride(lda, cute::Int<1>{}, sa),
                                 cute::make_stride(ldb, cute::Int<1>{}, sb), a, b, d, m, n, k, batch, workspace,
                                 workspace_bytes, s);
  }
  return PO_EINVAL;
}

}  // namespace

extern "C" {

#ifdef PO_PROBE_EXPORTS
int po_probe_gemm_smem(int variant) {
  switch (variant) {
    case 0: return (int)sizeof(typename RowRowT<PO_FASTF32_TILE_N>::Kernel::SharedStorage);
    case 1: return (int)sizeof(typename ColRowT<PO_FASTF32_TILE_N>::Kernel::SharedStorage);
    default: return (int)sizeof(typename RowColT<PO_FASTF32_TILE_N>::Kernel::SharedStorage);
  }
}
#endif

int po_set_gemm_tile(int32_t tile_n) {
  if (tile_n != 64 && tile_n != 128) return PO_EINVAL;
  g_tile_n = tile_n;
  return 0;
}

int po_get_gemm_tile(void) { return g_tile_n; }

int po_gemm_f32x3_available(void) { return 1; }

int po_gemm_f32x3(int32_t a_col_major, int32_t b_col_major, const float* a, int64_t lda, int64_t sa, const float* b,
                  int64_t ldb, int64_t sb, float* d, int64_t m, int64_t n, int64_t k, int64_t batch, void* workspace,
                  int64_t workspace_bytes, void* stream) {
  if (m < 1 || n < 1 || k < 1 || batch < 1 || a == nullptr || b == nullptr || d == nullptr) return PO_EINVAL;
  if (lda % kAlign || ldb % kAlign || n % kAlign || sa % kAlign || sb % kAlign) return PO_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (g_tile_n == 128)
    return dispatch_gemm<128>(a_col_major, b_col_major, a, lda, sa, b, ldb, sb, d, m, n, k, batch, workspace,
                              workspace_bytes, s);
  return dispatch_gemm<64>(a_col_major, b_col_major, a, lda, sa, b, ldb, sb, d, m, n, k, batch, workspace,
                           workspace_bytes, s);
}

}  // extern "C"
