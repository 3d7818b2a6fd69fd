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

namespace {

constexpr int kHeadThreads = 256;
constexpr int kHeadMaxC = 32;
constexpr int kGSmemFloats = 2048;  // g (rows x C) staged in shared memory up to 8 KB (static + dynamic <= 48 KB)

template <int CMAX>
__global__ void __launch_bounds__(kHeadThreads) head_fwd_kernel(const float* __restrict__ x, int64_t in,
                                                                const float* __restrict__ w,
                                                                const float* __restrict__ b, int C,
                                                                float* __restrict__ out, uint8_t* flags,
                                                                int64_t flag_index) {
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
  if (tid < C) {
    float s = part[0][tid];
#pragma unroll
    for (int q = 1; q < kHeadThreads / 32; ++q) s += part[q][tid];  // warp order
    const float o = (b != nullptr ? b[tid] : 0.f) + s;
    out[r * C + tid] = o;
    if (flags != nullptr && !isfinite(o)) flags[flag_index] = 0;
  }
}

template <int CMAX>
__global__ void __launch_bounds__(kHeadThreads) head_bwd_kernel(const float* __restrict__ x, int64_t rows,
                                                                int64_t in, const float* __restrict__ g, int C,
                                                                const float* __restrict__ w, float* __restrict__ dx,
                                                                float* __restrict__ dw, float* __restrict__ db,
                                                                int accumulate, int64_t dx_blocks) {
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

}  // namespace

extern "C" {

int po_head_supported(int64_t rows, int64_t in, int64_t classes) {
  return rows >= 1 && rows <= 0x7fffffff && in >= 1 && classes >= 1 && classes <= kHeadMaxC;
}

int po_head_fwd(const float* x, int64_t rows, int64_t in, const float* w, const float* b, int32_t classes,
                float* out, uint8_t* flags, int64_t flag_index, void* stream) {
  if (!po_head_supported(rows, in, classes) || x == nullptr || w == nullptr || out == nullptr || flag_index < 0)
    return PO_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid((unsigned)rows);
  switch (head_cmax(classes)) {
    case 8: head_fwd_kernel<8><<<grid, kHeadThreads, 0, s>>>(x, in, w, b, classes, out, flags, flag_index); break;
    case 16: head_fwd_kernel<16><<<grid, kHeadThreads, 0, s>>>(x, in, w, b, classes, out, flags, flag_index); break;
    default: head_fwd_kernel<32><<<grid, kHeadThreads, 0, s>>>(x, in, w, b, classes, out, flags, flag_index); break;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
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
      head_bwd_kernel<8><<<grid, kHeadThreads, smem, s>>>(x, rows, in, g, classes, w, dx, dw, db, accumulate,
                                                          dx_blocks);
      break;
    case 16:
      head_bwd_kernel<16><<<grid, kHeadThreads, smem, s>>>(x, rows, in, g, classes, w, dx, dw, db, accumulate,
                                                           dx_blocks);
      break;
    default:
      head_bwd_kernel<32><<<grid, kHeadThreads, smem, s>>>(x, rows, in, g, classes, w, dx, dw, db, accumulate,
                                                           dx_blocks);
      break;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
