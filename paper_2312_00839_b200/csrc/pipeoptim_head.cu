// pipeoptim_head.cu — the narrow output layer of an MLP pipeline's last stage
// (in -> C classes, C <= 32, linear activation: config 1's 1024 -> 10).
//
// The library GEMMs are built for wide outputs: at C = 10 the forward
// (x @ W + b, then the split-K reduce / bias epilogue) and the backward
// (dpre = g, db = colsum, dW = x^T g, dx = g W^T) take six latency-bound
// launches, ~40 us of serialised device time per mini-batch on config 1's
// single-GPU run (profiles/r1h_pipe_stage_streams_pred_on.txt). Here the
// forward is one launch (one CTA per row: each thread accumulates C partial
// dot products over its slice of the row, then a fixed-order reduction over
// the CTA) and the whole backward another (CTAs 0..rows-1 form the input
// gradient rows, the others the weight-gradient rows, the first of those
// also the bias gradient). Every sum runs in a fixed order: results are
// deterministic and identical across runners (stages.py:175-178, 200-208).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "pipeoptim.h"
#include "pipeoptim_pdl.cuh"

namespace {

constexpr int kHeadThreads = 256;
constexpr int kHeadMaxC = 32;
constexpr int kGSmemFloats = 2048;  // g (rows x C) staged in shared memory up to 8 KB (static + dynamic <= 48 KB)

// The reductions of loss_grad_kernel (pipeoptim_stage_ops.cu), restated so
// that the fused forward + loss below produces the same bits: a lane-xor
// butterfly inside each warp, then the warp totals in warp 0.
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < blockDim.x / 32) ? sh[threadIdx.x] : 0.f;
  if (w == 0) v = warp_sum(v);
  if (threadIdx.x == 0) sh[32] = v;
  __syncthreads();
  return sh[32];
}

// Loss inputs of the fused forward (LOSS = true): one-hot / regression
// targets (rows x C), the loss kind (PO_LOSS_*), dL/dout, the row partials +
// last-CTA counter (po_loss_grad's scratch layout) and the scalar loss.
struct LossArgs {
  const float* target;
  int kind;
  float* grad;
  float* row_part;
  unsigned int* counter;
  float* loss;
};

template <int CMAX, bool LOSS>
__global__ void __launch_bounds__(kHeadThreads) head_fwd_kernel(const float* __restrict__ x, int64_t rows,
                                                                int64_t in, const float* __restrict__ w,
                                                                const float* __restrict__ b, int C,
                                                                float* __restrict__ out, uint8_t* flags,
                                                                int64_t flag_index, LossArgs la) {
  pdl_wait();
  pdl_trigger();
  __shared__ float part[kHeadThreads / 32][CMAX];
  const int64_t r = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float acc[CMAX];
#pragma unroll
  for (int c = 0; c < CMAX; ++c) acc[c] = 0.f;
  for (int64_t i = tid; i < in; i += kHeadThreads) {
    const float xv = x[r * in + i];
    const float* wr = w + i * C;
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < C) acc[c] = fmaf(xv, wr[c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < CMAX; ++c) {
    float v = acc[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[warp][c] = v;
  }
  __syncthreads();
  float o = 0.f;
  if (tid < C) {
    float s = part[0][tid];
#pragma unroll
    for (int q = 1; q < kHeadThreads / 32; ++q) s += part[q][tid];  // warp order
    o = (b != nullptr ? b[tid] : 0.f) + s;
    out[r * C + tid] = o;
    if (flags != nullptr && !isfinite(o)) flags[flag_index] = 0;
  }
  if constexpr (LOSS) {
    // the row's C <= 32 logits sit in warp 0's lanes 0..C-1 (column c = lane
    // c, as in loss_grad_kernel); warps 1.. contribute exact zeros there
    __shared__ float sh[33];
    __shared__ bool last;
    if (warp == 0) {
      const bool on = tid < C;
      const float y = on ? la.target[r * C + tid] : 0.f;
      float* g = la.grad + r * C;
      float row;
      if (la.kind == PO_LOSS_SOFTMAX_XENT) {  // linalg.py:228-235
        float m = -INFINITY;
        if (on) m = fmaxf(m, o);
        m = warp_max(m);
        const float e = on ? expf(o - m) : 0.f;
        const float ssum = warp_sum(e);
        float picked = 0.f;
        if (on) {
          const float sm = expf(o - m) / ssum;
          picked = sm * y;
          g[tid] = (sm - y) * (1.0f / (float)rows);
        }
        row = -logf(warp_sum(picked));
      } else {  // mse, linalg.py:223-227
        float a = 0.f;
        if (on) {
          const float d = o - y;
          a = d * d;
          g[tid] = d * (2.0f / (float)(rows * C));
        }
        row = warp_sum(a);
      }
      if (tid == 0) {
        la.row_part[r] = row;
        __threadfence();
        last = atomicAdd(la.counter, 1u) == (unsigned int)(rows - 1);
      }
    }
    __syncthreads();
    if (last) {  // fixed-order reduction of the row partials (loss_grad_kernel's)
      __threadfence();
      float a = 0.f;
      for (int64_t i = tid; i < rows; i += kHeadThreads) a += ((volatile float*)la.row_part)[i];
      a = block_sum(a, sh);
      if (tid == 0) {
        *la.loss = (la.kind == PO_LOSS_SOFTMAX_XENT) ? a / (float)rows : a / (float)(rows * C);
        *la.counter = 0u;  // re-armed for the next launch (graph replays)
      }
    }
  }
}

template <int CMAX>
__global__ void __launch_bounds__(kHeadThreads) head_bwd_kernel(const float* __restrict__ x, int64_t rows,
                                                                int64_t in, const float* __restrict__ g, int C,
                                                                const float* __restrict__ w, float* __restrict__ dx,
                                                                float* __restrict__ dw, float* __restrict__ db,
                                                                int accumulate, int64_t dx_blocks) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float gs[];  // g (rows x C) when it fits, else one row
  const int tid = threadIdx.x;
  if ((int64_t)blockIdx.x < dx_blocks) {
    // input gradient row r: dx[r][i] = sum_c g[r][c] w[i][c] (live weights, S9)
    const int64_t r = blockIdx.x;
    if (tid < C) gs[tid] = g[r * C + tid];
    __syncthreads();
    for (int64_t i = tid; i < in; i += kHeadThreads) {
      const float* wr = w + i * C;
      float s = 0.f;
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < C) s = fmaf(gs[c], wr[c], s);
      dx[r * in + i] = s;
    }
    return;
  }
  // weight-gradient rows i of this CTA (32 of them, one per lane):
  // dw[i][c] = sum_r x[r][i] g[r][c]; warp q takes rows r = q, q + 8, ...
  // (loads coalesced along i, four rows in flight), then the 8 warp
  // partials are summed in warp order through shared memory
  const int64_t blk = (int64_t)blockIdx.x - dx_blocks;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kHeadThreads / 32;
  const bool staged = rows * C <= kGSmemFloats;
  if (staged) {
    for (int64_t k = tid; k < rows * C; k += kHeadThreads) gs[k] = g[k];
    __syncthreads();
  }
  const float* gg = staged ? gs : g;
  const int64_t i = blk * 32 + lane;
  float acc[CMAX];
#pragma unroll
  for (int c = 0; c < CMAX; ++c) acc[c] = 0.f;
  if (i < in) {
    int64_t r = warp;
    for (; r + 3 * kWarps < rows; r += 4 * kWarps) {
      float xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = x[(r + u * kWarps) * in + i];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < C) acc[c] = fmaf(xv[u], gg[(r + u * kWarps) * C + c], acc[c]);
    }
    for (; r < rows; r += kWarps) {
      const float xv = x[r * in + i];
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < C) acc[c] = fmaf(xv, gg[r * C + c], acc[c]);
    }
  }
  __shared__ float part[kWarps][32][CMAX + 1];
#pragma unroll
  for (int c = 0; c < CMAX; ++c) part[warp][lane][c] = acc[c];
  __syncthreads();
  for (int k = tid; k < 32 * C; k += kHeadThreads) {
    const int l = k / C, c = k % C;
    const int64_t ii = blk * 32 + l;
    if (ii < in) {
      float v = part[0][l][c];
#pragma unroll
      for (int q = 1; q < kWarps; ++q) v += part[q][l][c];  // warp order
      dw[ii * C + c] = accumulate ? dw[ii * C + c] + v : v;
    }
  }
  if (blk == 0 && tid < C) {  // bias gradient: column sums in row order
    float v = 0.f;
    for (int64_t r = 0; r < rows; ++r) v += gg[r * C + tid];
    db[tid] = accumulate ? db[tid] + v : v;
  }
}

int head_cmax(int C) { return C <= 8 ? 8 : C <= 16 ? 16 : 32; }

template <bool LOSS>
int launch_head_fwd(const float* x, int64_t rows, int64_t in, const float* w, const float* b, int32_t classes,
                    float* out, uint8_t* flags, int64_t flag_index, LossArgs la, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid((unsigned)rows);
  switch (head_cmax(classes)) {
    case 8:
      pdl_launch(head_fwd_kernel<8, LOSS>, grid, dim3(kHeadThreads), 0, s, x, rows, in, w, b, classes, out, flags,
                 flag_index, la);
      break;
    case 16:
      pdl_launch(head_fwd_kernel<16, LOSS>, grid, dim3(kHeadThreads), 0, s, x, rows, in, w, b, classes, out, flags,
                 flag_index, la);
      break;
    default:
      pdl_launch(head_fwd_kernel<32, LOSS>, grid, dim3(kHeadThreads), 0, s, x, rows, in, w, b, classes, out, flags,
                 flag_index, la);
      break;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // namespace

extern "C" {

int po_head_supported(int64_t rows, int64_t in, int64_t classes) {
  return rows >= 1 && rows <= 0x7fffffff && in >= 1 && classes >= 1 && classes <= kHeadMaxC;
}

int po_head_fwd(const float* x, int64_t rows, int64_t in, const float* w, const float* b, int32_t classes,
                float* out, uint8_t* flags, int64_t flag_index, void* stream) {
  if (!po_head_supported(rows, in, classes) || x == nullptr || w == nullptr || out == nullptr || flag_index < 0)
    return PO_EINVAL;
  return launch_head_fwd<false>(x, rows, in, w, b, classes, out, flags, flag_index, LossArgs{}, stream);
}

int po_head_fwd_loss(const float* x, int64_t rows, int64_t in, const float* w, const float* b, int32_t classes,
                     const float* target, int32_t kind, float* out, float* grad, float* loss, float* scratch,
                     uint8_t* flags, int64_t flag_index, void* stream) {
  if (!po_head_supported(rows, in, classes) || x == nullptr || w == nullptr || out == nullptr || flag_index < 0)
    return PO_EINVAL;
  if ((kind != PO_LOSS_MSE && kind != PO_LOSS_SOFTMAX_XENT) || target == nullptr || grad == nullptr ||
      loss == nullptr || scratch == nullptr)
    return PO_EINVAL;
  // scratch: po_loss_grad's layout ([rows] row partials, then a uint32 counter zeroed once)
  const LossArgs la{target, kind, grad, scratch, reinterpret_cast<unsigned int*>(scratch + rows), loss};
  return launch_head_fwd<true>(x, rows, in, w, b, classes, out, flags, flag_index, la, stream);
}

int po_head_bwd(const float* x, int64_t rows, int64_t in, const float* g, int32_t classes, const float* w, float* dx,
                float* dw, float* db, int32_t accumulate, void* stream) {
  if (!po_head_supported(rows, in, classes) || x == nullptr || g == nullptr || w == nullptr || dw == nullptr ||
      db == nullptr)
    return PO_EINVAL;
  const int64_t dx_blocks = dx != nullptr ? rows : 0;
  const int64_t dw_blocks = (in + 31) / 32;
  if (dx_blocks + dw_blocks > 0x7fffffff) return PO_EINVAL;
  const size_t smem = (size_t)(rows * classes <= kGSmemFloats ? rows * classes : classes) * sizeof(float);
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid((unsigned)(dx_blocks + dw_blocks));
  switch (head_cmax(classes)) {
    case 8:
      pdl_launch(head_bwd_kernel<8>, grid, dim3(kHeadThreads), smem, s, x, rows, in, g, classes, w, dx, dw, db,
                 accumulate, dx_blocks);
      break;
    case 16:
      pdl_launch(head_bwd_kernel<16>, grid, dim3(kHeadThreads), smem, s, x, rows, in, g, classes, w, dx, dw, db,
                 accumulate, dx_blocks);
      break;
    default:
      pdl_launch(head_bwd_kernel<32>, grid, dim3(kHeadThreads), smem, s, x, rows, in, g, classes, w, dx, dw, db,
                 accumulate, dx_blocks);
      break;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
