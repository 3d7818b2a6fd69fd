// pipeoptim_stage_ops.cu — fused per-event stage ops for the 1F1B runners.
//
// The runners' small per-event ops were each several torch launches
// (profiles/r1_pipeline_breakdown.md): a finiteness check of a forward output
// (isfinite -> abs/compare/and -> all-reduce -> index copy: 5 launches) and
// the last stage's loss + gradient (~10 launches). Here each is ONE launch:
//
//   po_all_finite   flags[index] = 0 if any x is NaN/Inf (flags pre-set to 1).
//                   Replaces stages.py:182's require_finite in deferred mode.
//   po_loss_grad    softmax cross-entropy or MSE loss AND its gradient
//                   (linalg.py:212-241), the loss reduced in a fixed order by
//                   the last CTA to finish (deterministic, no float atomics).
//   po_splitk_bias_act  the reduction of a split-K GEMM (S partial products
//                   summed in a fixed order) fused with the layer's bias and
//                   activation — the config-1 GEMMs have M = batch = 128 rows and
//                   a long K, so cuBLAS runs them on a handful of output tiles;
//                   split-K bmm + this kernel is 2-3x faster (scripts/gemm_splitk.py)
//   po_relu_bwd_bias  a ReLU layer's backward elementwise part AND its bias
//                   gradient: dpre = g * (h > 0), db (+)= colsum(dpre)
//                   (stages.py:200-206) — replaces compare + multiply +
//                   column-sum (3 launches, dpre written then re-read); g may
//                   arrive as the split-K partials of the next layer's input
//                   gradient, summed here in a fixed order.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "pipeoptim.h"
#include "pipeoptim_pdl.cuh"

namespace {

__global__ void all_finite_kernel(const float* __restrict__ x, int64_t n, uint8_t* flags, int64_t index) {
  pdl_wait();
  pdl_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n4 = (reinterpret_cast<uintptr_t>(x) % 16 == 0) ? n / 4 : 0;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (int64_t j = i; j < n4; j += stride) {
    float4 v = x4[j];
    bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
  }
  for (int64_t j = n4 * 4 + i; j < n; j += stride) bad |= !isfinite(x[j]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flags[index] = 0;
}

constexpr int kLossThreads = 256;

__device__ __forceinline__ float block_reduce_max(float v, float* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < blockDim.x / 32) ? sh[threadIdx.x] : -INFINITY;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (threadIdx.x == 0) sh[32] = v;
  __syncthreads();
  return sh[32];
}

__device__ __forceinline__ float block_reduce_sum(float v, float* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < blockDim.x / 32) ? sh[threadIdx.x] : 0.f;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x == 0) sh[32] = v;
  __syncthreads();
  return sh[32];
}

// One CTA per row. softmax_xent: z = x - max; e = exp(z); sm = e / sum(e);
// row loss = -log(sum(sm * y)); grad = (sm - y) / rows. mse: row partial
// sum of (x - y)^2; grad = 2 (x - y) / numel. The last CTA reduces the row
// partials in row order into *loss.
__global__ void loss_grad_kernel(const float* __restrict__ pred, const float* __restrict__ target, int64_t rows,
                                 int64_t cols, int kind, float* __restrict__ grad, float* __restrict__ row_part,
                                 unsigned int* counter, float* loss) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sh[33];
  __shared__ bool last;
  const int64_t r = blockIdx.x;
  const float* x = pred + r * cols;
  const float* y = target + r * cols;
  float* g = grad + r * cols;
  float part;
  if (kind == 1) {  // softmax cross-entropy (linalg.py:228-235)
    float m = -INFINITY;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) m = fmaxf(m, x[c]);
    m = block_reduce_max(m, sh);
    float s = 0.f;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) s += expf(x[c] - m);
    s = block_reduce_sum(s, sh);
    float picked = 0.f;
    const float inv_rows = 1.0f / (float)rows;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const float sm = expf(x[c] - m) / s;
      picked += sm * y[c];
      g[c] = (sm - y[c]) * inv_rows;
    }
    picked = block_reduce_sum(picked, sh);
    part = -logf(picked);
  } else {  // mse (linalg.py:223-227)
    const float scale = 2.0f / (float)(rows * cols);
    float acc = 0.f;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const float d = x[c] - y[c];
      acc += d * d;
      g[c] = d * scale;
    }
    part = block_reduce_sum(acc, sh);
  }
  if (threadIdx.x == 0) {
    row_part[r] = part;
    __threadfence();
    last = atomicAdd(counter, 1u) == (unsigned int)(rows - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    // fixed-order reduction of the row partials by the last CTA
    float acc = 0.f;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) acc += ((volatile float*)row_part)[i];
    acc = block_reduce_sum(acc, sh);
    if (threadIdx.x == 0) {
      *loss = (kind == 1) ? acc / (float)rows : acc / (float)(rows * cols);
      *counter = 0u;  // re-armed for the next launch (graph replays)
    }
  }
}

// One CTA per 8 columns: thread t handles column t % 8 and rows t / 8,
// t / 8 + 64, ... (a warp reads 4 rows x 32 contiguous bytes per load), keeps
// its column partial in a register, then the 64 row-lanes' partials of each
// column are summed in row-lane order through shared memory: a fixed
// reduction order, so the bias gradient is deterministic. 8-column CTAs put
// 128 CTAs on a 1024-wide layer; the up-to-8 split-K partials of an element
// are loaded together (independent loads in flight), then summed in order.
constexpr int kReluCols = 8, kReluLanes = 64;

// g: `splits` partial products [splits x rows x cols], summed in order 0..S-1.
// g and dpre may alias when splits == 1 (each element is read, then written,
// by one thread)
__global__ void relu_bwd_bias_kernel(const float* g, int splits, const float* __restrict__ h, int64_t rows,
                                     int64_t cols, float* dpre, float* __restrict__ db, int accumulate, int mask) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = rows * cols;
  __shared__ float part[kReluLanes][kReluCols];
  const int cl = threadIdx.x % kReluCols, lane = threadIdx.x / kReluCols;
  const int64_t c = (int64_t)blockIdx.x * kReluCols + cl;
  float acc = 0.f;
  if (c < cols) {
    for (int64_t r = lane; r < rows; r += kReluLanes) {
      const int64_t i = r * cols + c;
      float v[8];
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < splits) v[s] = g[(int64_t)s * n + i];
      const bool keep = !mask || h[i] > 0.f;  // g * (pre > 0): relu(pre) > 0 <=> pre > 0
      float gi = v[0];
#pragma unroll
      for (int s = 1; s < 8; ++s)
        if (s < splits) gi += v[s];
      for (int s = 8; s < splits; ++s) gi += g[(int64_t)s * n + i];
      const float o = keep ? gi : 0.f;
      dpre[i] = o;
      acc += o;
    }
  }
  part[lane][cl] = acc;
  __syncthreads();
  if (lane == 0 && c < cols) {
    float s = 0.f;
#pragma unroll 8
    for (int k = 0; k < kReluLanes; ++k) s += part[k][cl];
    db[c] = accumulate ? db[c] + s : s;
  }
}

// out[i] = act(sum_s part[s*n + i] + bias[i % cols]), s in order 0..S-1;
// pre_out (nullable) receives the pre-activation. act: 0 linear, 1 relu, 2 tanh.
// flags (nullable): flags[flag_index] = 0 if any output is NaN/Inf — the
// stage-output finiteness check (stages.py:182) folded into the epilogue.
__device__ __forceinline__ float act_fn(float x, int act) {
  return act == 1 ? (x > 0.f ? x : 0.f) : act == 2 ? tanhf(x) : x;
}

template <bool VEC4>
__global__ void splitk_bias_act_kernel(const float* __restrict__ part, int S, int64_t n, int64_t cols,
                                       const float* __restrict__ bias, int act, float* __restrict__ out,
                                       float* __restrict__ pre_out, uint8_t* flags, int64_t flag_index) {
  pdl_wait();
  pdl_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  if constexpr (VEC4) {
    const int64_t n4 = n / 4;
    const float4* p4 = reinterpret_cast<const float4*>(part);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      // up to 8 partials' loads issued together, then summed in order 0..S-1
      float4 v[8];
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < S) v[s] = p4[(int64_t)s * n4 + i];
      float4 acc = v[0];
#pragma unroll
      for (int s = 1; s < 8; ++s)
        if (s < S) {
          acc.x += v[s].x;
          acc.y += v[s].y;
          acc.z += v[s].z;
          acc.w += v[s].w;
        }
      for (int s = 8; s < S; ++s) {
        const float4 a = p4[(int64_t)s * n4 + i];
        acc.x += a.x;
        acc.y += a.y;
        acc.z += a.z;
        acc.w += a.w;
      }
      if (bias != nullptr) {
        const float4 bv = reinterpret_cast<const float4*>(bias)[(i * 4 % cols) / 4];
        acc.x += bv.x;
        acc.y += bv.y;
        acc.z += bv.z;
        acc.w += bv.w;
      }
      if (pre_out != nullptr) reinterpret_cast<float4*>(pre_out)[i] = acc;
      float4 o = make_float4(act_fn(acc.x, act), act_fn(acc.y, act), act_fn(acc.z, act), act_fn(acc.w, act));
      reinterpret_cast<float4*>(out)[i] = o;
      bad |= !isfinite(o.x) | !isfinite(o.y) | !isfinite(o.z) | !isfinite(o.w);
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      float acc = part[i];
      for (int s = 1; s < S; ++s) acc += part[(int64_t)s * n + i];
      if (bias != nullptr) acc += bias[i % cols];
      if (pre_out != nullptr) pre_out[i] = acc;
      const float o = act_fn(acc, act);
      out[i] = o;
      bad |= !isfinite(o);
    }
  }
  if (flags != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flags[flag_index] = 0;
}

int sm_count_ops() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

}  // namespace

extern "C" {

int po_act_bwd_bias(int32_t act, const float* g, int32_t splits, const float* h, int64_t rows, int64_t cols,
                    float* dpre, float* db, int32_t accumulate, void* stream);

// Invalidate the L2 lines of a dead buffer WITHOUT writing them back
// (discard.global.L2): a predicted-weights staging buffer after the forward
// that consumed it, or a gradient after the update that consumed it, would
// otherwise cost an HBM write-back of data nobody reads again. Only whole
// 128-byte lines inside [p, p + bytes) are discarded; their memory contents
// become unspecified.
__global__ void l2_discard_kernel(char* base, int64_t lines) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < lines; i += stride)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + i * 128) : "memory");
}

int po_l2_discard(void* p, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && p == nullptr)) return PO_EINVAL;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t lo = (a + 127) & ~uintptr_t(127);
  const uintptr_t hi = (a + (uintptr_t)bytes) & ~uintptr_t(127);
  if (hi <= lo) return 0;
  const int64_t lines = (int64_t)((hi - lo) / 128);
  static int sms = 0;
  if (sms == 0) sms = sm_count_ops();
  const int block = 256;
  int64_t grid = (lines + block - 1) / block;
  if (grid > 4 * sms) grid = 4 * sms;
  l2_discard_kernel<<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(reinterpret_cast<char*>(lo), lines);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

int po_all_finite(const float* x, int64_t n, uint8_t* flags, int64_t index, void* stream) {
  if (n < 0 || flags == nullptr || index < 0 || (n > 0 && x == nullptr)) return PO_EINVAL;
  if (n == 0) return 0;
  static int sms = 0;
  if (sms == 0) sms = sm_count_ops();
  const int block = 256;
  int64_t want = (n / 4 + block - 1) / block;
  int64_t grid = want < 1 ? 1 : (want > 4 * sms ? 4 * sms : want);
  pdl_launch(all_finite_kernel, dim3((unsigned)grid), dim3(block), 0, (cudaStream_t)stream, x, n, flags, index);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

int po_splitk_bias_act(const float* part, int32_t splits, int64_t rows, int64_t cols, const float* bias,
                       int32_t act, float* out, float* pre_out, uint8_t* flags, int64_t flag_index, void* stream) {
  if (splits < 1 || rows < 0 || cols < 1 || act < 0 || act > 2 || out == nullptr || (rows > 0 && part == nullptr) ||
      flag_index < 0)
    return PO_EINVAL;
  const int64_t n = rows * cols;
  if (n == 0) return 0;
  static int sms = 0;
  if (sms == 0) sms = sm_count_ops();
  const int block = 128;  // a 128 x 1024 output is 256 CTAs: every SM gets work
  const bool vec = cols % 4 == 0 && ((reinterpret_cast<uintptr_t>(part) | reinterpret_cast<uintptr_t>(out) |
                                      reinterpret_cast<uintptr_t>(pre_out) | reinterpret_cast<uintptr_t>(bias)) &
                                     15) == 0;
  int64_t want = ((vec ? n / 4 : n) + block - 1) / block;
  const int64_t grid = want > 8 * sms ? 8 * sms : want;
  if (vec)
    pdl_launch(splitk_bias_act_kernel<true>, dim3((unsigned)grid), dim3(block), 0, (cudaStream_t)stream, part, splits, n,
               cols, bias, act, out, pre_out, flags, flag_index);
  else
    pdl_launch(splitk_bias_act_kernel<false>, dim3((unsigned)grid), dim3(block), 0, (cudaStream_t)stream, part, splits,
               n, cols, bias, act, out, pre_out, flags, flag_index);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

int po_relu_bwd_bias(const float* g, int32_t splits, const float* h, int64_t rows, int64_t cols, float* dpre,
                     float* db, int32_t accumulate, void* stream) {
  return po_act_bwd_bias(1, g, splits, h, rows, cols, dpre, db, accumulate, stream);
}

int po_act_bwd_bias(int32_t act, const float* g, int32_t splits, const float* h, int64_t rows, int64_t cols,
                    float* dpre, float* db, int32_t accumulate, void* stream) {
  if (rows < 0 || cols < 0 || splits < 1 || (act != 0 && act != 1)) return PO_EINVAL;
  if (rows == 0 || cols == 0) {
    if (cols > 0 && !accumulate && db != nullptr) {
      cudaError_t e = cudaMemsetAsync(db, 0, (size_t)cols * sizeof(float), (cudaStream_t)stream);
      return e == cudaSuccess ? 0 : (int)e;
    }
    return 0;
  }
  if (g == nullptr || (act == 1 && h == nullptr) || dpre == nullptr || db == nullptr) return PO_EINVAL;
  const int64_t grid = (cols + kReluCols - 1) / kReluCols;
  if (grid > 0x7fffffff) return PO_EINVAL;
  pdl_launch(relu_bwd_bias_kernel, dim3((unsigned)grid), dim3(kReluCols * kReluLanes), 0, (cudaStream_t)stream, g,
             splits, h, rows, cols, dpre, db, accumulate, act);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

int po_loss_grad(int32_t kind, const float* pred, const float* target, int64_t rows, int64_t cols, float* grad,
                 float* loss, float* scratch, void* stream) {
  if ((kind != PO_LOSS_MSE && kind != PO_LOSS_SOFTMAX_XENT) || rows < 1 || cols < 1) return PO_EINVAL;
  if (pred == nullptr || target == nullptr || grad == nullptr || loss == nullptr || scratch == nullptr)
    return PO_EINVAL;
  if (rows > 0x7fffffff) return PO_EINVAL;
  // scratch layout: [rows] float row partials, then one uint32 counter (caller zeroes it once)
  unsigned int* counter = reinterpret_cast<unsigned int*>(scratch + rows);
  pdl_launch(loss_grad_kernel, dim3((unsigned)rows), dim3(kLossThreads), 0, (cudaStream_t)stream, pred, target, rows,
             cols, kind, grad, scratch, counter, loss);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
