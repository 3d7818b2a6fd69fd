// pipeoptim_lstm.cu — LSTM cell kernels for the live-weight GNMT stages.
//
// The reference's stage semantics (stages.py:187-209): the
// forward runs on the policy's weights (W_hat when predicted) and stashes its
// activations; the backward multiplies by the LIVE weights for the input
// gradient and forms dW from the stashed activations. cuDNN's LSTM keeps its
// own packed copy of the forward weights, so it cannot back-propagate through
// different weights. stage_models.LiveLSTM therefore runs the recurrence as
// cuBLAS GEMMs (gates_t += h_{t-1} W_hh^T, dh_{t-1} = dgates_t W_hh_live) and
// these two elementwise kernels, one launch per time step each:
//
//   po_lstm_cell_fwd  gate nonlinearities, c_t, h_t (PyTorch gate order i,f,g,o);
//                     the activations overwrite the pre-activations in place
//                     (the backward's stash), h_t is written time-major (next
//                     step's GEMM operand, dW_hh's operand) and, optionally,
//                     batch-first into the layer output (no transpose pass).
//   po_lstm_cell_bwd  dh = dy_t + dh_rec; the cell's chain rule; writes the
//                     pre-activation gradients dgates_t and carries dc.
//
// Both are HBM/L2 streams of a few hundred KB per step (B x 4H floats), so
// they are latency-bound: 128-bit accesses, one thread per 4 hidden units of
// one batch row, one wave.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "pipeoptim.h"

namespace {

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

#define PO_MAP4(out, a, expr)                                                                     \
  do {                                                                                            \
    { const float x = (a).x; (out).x = (expr); }                                                  \
    { const float x = (a).y; (out).y = (expr); }                                                  \
    { const float x = (a).z; (out).z = (expr); }                                                  \
    { const float x = (a).w; (out).w = (expr); }                                                  \
  } while (0)

// thread -> (row b, hidden units j..j+3); hidden % 4 == 0, rows 16-byte aligned
__device__ __forceinline__ void add4(float4& a, const float4 b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// rec (nullable): `splits` partial products [splits x batch x 4*hidden] of
// h_{t-1} W_hh^T (a split-K GEMM), added to the pre-activations in order.
__global__ void lstm_cell_fwd_kernel(float* __restrict__ gates, const float* __restrict__ rec, int splits,
                                     const float* __restrict__ c_prev, float* __restrict__ c_out,
                                     float* __restrict__ h_out, float* __restrict__ y_out, int64_t y_ld,
                                     int64_t batch, int64_t hidden) {
  const int64_t q = hidden / 4;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * q) return;
  const int64_t b = idx / q, j = (idx - b * q) * 4;
  float* gr = gates + b * 4 * hidden;
  float4 ai = ld4(gr + j), af = ld4(gr + hidden + j), ag = ld4(gr + 2 * hidden + j), ao = ld4(gr + 3 * hidden + j);
  if (rec != nullptr) {
    float4 si = ld4(rec + b * 4 * hidden + j), sf = ld4(rec + b * 4 * hidden + hidden + j),
           sg = ld4(rec + b * 4 * hidden + 2 * hidden + j), so = ld4(rec + b * 4 * hidden + 3 * hidden + j);
    for (int s = 1; s < splits; ++s) {
      const float* rs = rec + (int64_t)s * batch * 4 * hidden + b * 4 * hidden;
      add4(si, ld4(rs + j));
      add4(sf, ld4(rs + hidden + j));
      add4(sg, ld4(rs + 2 * hidden + j));
      add4(so, ld4(rs + 3 * hidden + j));
    }
    add4(ai, si);
    add4(af, sf);
    add4(ag, sg);
    add4(ao, so);
  }
  float4 i, f, g, o;
  PO_MAP4(i, ai, sigmoidf_(x));
  PO_MAP4(f, af, sigmoidf_(x));
  PO_MAP4(g, ag, tanhf(x));
  PO_MAP4(o, ao, sigmoidf_(x));
  const float4 cp = c_prev ? ld4(c_prev + b * hidden + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 c, h;
  c.x = f.x * cp.x + i.x * g.x;
  c.y = f.y * cp.y + i.y * g.y;
  c.z = f.z * cp.z + i.z * g.z;
  c.w = f.w * cp.w + i.w * g.w;
  h.x = o.x * tanhf(c.x);
  h.y = o.y * tanhf(c.y);
  h.z = o.z * tanhf(c.z);
  h.w = o.w * tanhf(c.w);
  st4(gr + j, i);
  st4(gr + hidden + j, f);
  st4(gr + 2 * hidden + j, g);
  st4(gr + 3 * hidden + j, o);
  st4(c_out + b * hidden + j, c);
  st4(h_out + b * hidden + j, h);
  if (y_out) st4(y_out + b * y_ld + j, h);
}

// dh_rec (nullable): `splits` partial products [splits x batch x hidden] of
// dgates_{t+1} W_hh (a split-K GEMM), summed in order.
__global__ void lstm_cell_bwd_kernel(const float* __restrict__ act, const float* __restrict__ c_prev,
                                     const float* __restrict__ c_cur, const float* __restrict__ dy, int64_t dy_ld,
                                     const float* __restrict__ dh_rec, int splits, float* __restrict__ dc,
                                     float* __restrict__ dgates, int64_t batch, int64_t hidden) {
  const int64_t q = hidden / 4;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * q) return;
  const int64_t b = idx / q, j = (idx - b * q) * 4;
  const float* ar = act + b * 4 * hidden;
  const float4 i = ld4(ar + j), f = ld4(ar + hidden + j), g = ld4(ar + 2 * hidden + j), o = ld4(ar + 3 * hidden + j);
  const int64_t e = b * hidden + j;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 c = ld4(c_cur + e);
  const float4 cp = c_prev ? ld4(c_prev + e) : z;
  const float4 y = dy ? ld4(dy + b * dy_ld + j) : z;
  float4 r = dh_rec ? ld4(dh_rec + e) : z;
  if (dh_rec != nullptr)
    for (int s = 1; s < splits; ++s) add4(r, ld4(dh_rec + (int64_t)s * batch * hidden + e));
  const float4 dcin = ld4(dc + e);
  float4 dcp, dai, daf, dag, dao;
#define PO_LSTM_BWD(k)                                                         \
  {                                                                            \
    const float dh = y.k + r.k;                                                \
    const float tc = tanhf(c.k);                                               \
    const float dct = dcin.k + dh * o.k * (1.0f - tc * tc);                    \
    dao.k = dh * tc * o.k * (1.0f - o.k);                                      \
    dai.k = dct * g.k * i.k * (1.0f - i.k);                                    \
    daf.k = dct * cp.k * f.k * (1.0f - f.k);                                   \
    dag.k = dct * i.k * (1.0f - g.k * g.k);                                    \
    dcp.k = dct * f.k;                                                         \
  }
  PO_LSTM_BWD(x) PO_LSTM_BWD(y) PO_LSTM_BWD(z) PO_LSTM_BWD(w)
#undef PO_LSTM_BWD
  float* dr = dgates + b * 4 * hidden;
  st4(dr + j, dai);
  st4(dr + hidden + j, daf);
  st4(dr + 2 * hidden + j, dag);
  st4(dr + 3 * hidden + j, dao);
  st4(dc + e, dcp);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

extern "C" {

int po_lstm_cell_fwd_sk(float* gates, const float* rec, int32_t splits, const float* c_prev, float* c_out,
                        float* h_out, float* y_out, int64_t y_ld, int64_t batch, int64_t hidden, void* stream);
int po_lstm_cell_bwd_sk(const float* act, const float* c_prev, const float* c, const float* dy, int64_t dy_ld,
                        const float* dh_rec, int32_t splits, float* dc, float* dgates, int64_t batch, int64_t hidden,
                        void* stream);

int po_lstm_cell_fwd(float* gates, const float* c_prev, float* c_out, float* h_out, float* y_out, int64_t y_ld,
                     int64_t batch, int64_t hidden, void* stream) {
  return po_lstm_cell_fwd_sk(gates, nullptr, 0, c_prev, c_out, h_out, y_out, y_ld, batch, hidden, stream);
}

int po_lstm_cell_fwd_sk(float* gates, const float* rec, int32_t splits, const float* c_prev, float* c_out,
                        float* h_out, float* y_out, int64_t y_ld, int64_t batch, int64_t hidden, void* stream) {
  if (batch < 1 || hidden < 4 || hidden % 4 != 0 || gates == nullptr || c_out == nullptr || h_out == nullptr ||
      (rec != nullptr && (splits < 1 || !aligned16(rec))))
    return PO_EINVAL;
  if (!aligned16(gates) || !aligned16(c_out) || !aligned16(h_out) || (c_prev && !aligned16(c_prev)) ||
      (y_out && (!aligned16(y_out) || y_ld % 4 != 0 || y_ld < hidden)))
    return PO_EINVAL;
  const int64_t threads = batch * (hidden / 4);
  const int block = 256;
  lstm_cell_fwd_kernel<<<(unsigned)((threads + block - 1) / block), block, 0, (cudaStream_t)stream>>>(
      gates, rec, splits, c_prev, c_out, h_out, y_out, y_ld, batch, hidden);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

int po_lstm_cell_bwd(const float* act, const float* c_prev, const float* c, const float* dy, int64_t dy_ld,
                     const float* dh_rec, float* dc, float* dgates, int64_t batch, int64_t hidden, void* stream) {
  return po_lstm_cell_bwd_sk(act, c_prev, c, dy, dy_ld, dh_rec, 1, dc, dgates, batch, hidden, stream);
}

int po_lstm_cell_bwd_sk(const float* act, const float* c_prev, const float* c, const float* dy, int64_t dy_ld,
                        const float* dh_rec, int32_t splits, float* dc, float* dgates, int64_t batch, int64_t hidden,
                        void* stream) {
  if (batch < 1 || hidden < 4 || hidden % 4 != 0 || act == nullptr || c == nullptr || dc == nullptr ||
      dgates == nullptr || (dh_rec != nullptr && splits < 1))
    return PO_EINVAL;
  if (!aligned16(act) || !aligned16(c) || !aligned16(dc) || !aligned16(dgates) || (c_prev && !aligned16(c_prev)) ||
      (dh_rec && !aligned16(dh_rec)) || (dy && (!aligned16(dy) || dy_ld % 4 != 0 || dy_ld < hidden)))
    return PO_EINVAL;
  const int64_t threads = batch * (hidden / 4);
  const int block = 256;
  lstm_cell_bwd_kernel<<<(unsigned)((threads + block - 1) / block), block, 0, (cudaStream_t)stream>>>(
      act, c_prev, c, dy, dy_ld, dh_rec, splits, dc, dgates, batch, hidden);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
