// pipeoptim_kernels.cu — sm_100a kernels + C-ABI for PipeOptim's
// optimizer-dependent weight prediction (arXiv 2312.00839, Eq. (5)) and the
// SGDM / Adam / AdamW update rules of the reference simulator
// (/root/reference/pkg/src/pipesim/optim.py).
//
// Everything here is an HBM-bound elementwise stream over flat fp32 per-stage
// buffers: no data reuse, ~1 flop/byte, so the design is the
// streaming one — 128/256-bit vector LDG/STG (LDG.E.128 / LDG.E.256 on
// sm_100a), a persistent grid sized in multiples of the SM count, several
// independent vector loads in flight per thread before any use, streaming cache
// hints so the 126 MB L2 is not polluted by data touched once, and the
// optimizer step + next-forward prediction fused into ONE pass (K3), so each
// parameter byte is read once per micro-step.
//
// Per-parameter algorithmic bytes (fp32):      SGDM   Adam/AdamW
//   K1 predict       (r W,state  w W_hat)       12      16
//   K2 step          (r W,g,state w W,state)     20      28
//   K3 step+predict  (K2 + w W_hat)              24      32
//
// Numerics follow the reference formulas in fp32 with IEEE div/sqrt (no
// fast-math): see Appendix A of SURVEY.md and the per-line citations below.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <string.h>

#include "pipeoptim.h"
#include "pipeoptim_rules.cuh"
#include "pipeoptim_pdl.cuh"

namespace {

struct Args {
  float* w;            // live weights (read, or read+write for steps)
  const float* g;      // gradient (read only)
  float* s1;           // sgdm momentum buffer | adam exp_avg | axpy direction
  float* s2;           // adam exp_avg_sq
  float* out;          // w_hat or dir_out
  int64_t n;
  unsigned long long* bad;  // smallest non-finite flat index (atomicMin)
  const po_coef* dc;   // nullable: per-launch scalars read from device memory
                       // (CUDA-graph replays), overriding c.{lr,c_pred,ibc1,ibc2}
  Coef c;
};

// The launch's coefficients: by value, or — for graph-captured launches whose
// step count / learning rate change between replays — from a device po_coef
// the host refreshes before each replay.
__device__ __forceinline__ Coef load_coef(const Args& a) {
  Coef c = a.c;
  if (a.dc != nullptr) {
    const po_coef d = *a.dc;
    c.lr = d.lr;
    c.c_pred = d.c_pred;
    c.ibc1 = d.inv_bc1;
    c.ibc2 = d.inv_bc2;
  }
  return c;
}

__host__ __device__ constexpr bool uses_w(int mode) {
  return mode == MODE_STEP || mode == MODE_STEP_DIR || mode == MODE_PREDICT ||
         mode == MODE_PREDICT_ZERO || mode == MODE_STEP_PREDICT || mode == MODE_AXPY;
}
__host__ __device__ constexpr bool writes_w(int mode) {
  return mode == MODE_STEP || mode == MODE_STEP_DIR || mode == MODE_STEP_PREDICT;
}
__host__ __device__ constexpr bool uses_g(int mode) { return writes_w(mode); }
__host__ __device__ constexpr bool uses_s1(int mode) {
  return mode == MODE_STEP || mode == MODE_STEP_DIR || mode == MODE_PREDICT ||
         mode == MODE_STEP_PREDICT || mode == MODE_DIRECTION || mode == MODE_AXPY;
}
__host__ __device__ constexpr bool uses_s2(int kind, int mode) {
  return kind != PO_SGDM && mode != MODE_AXPY && uses_s1(mode);
}
__host__ __device__ constexpr bool writes_state(int mode) { return writes_w(mode); }
#ifdef PO_PROBE_K3_NO_WHAT  // timing probe only (scripts/k3_no_what_probe.py): K3 skips its W_hat store
__host__ __device__ constexpr bool writes_out(int mode) { return mode != MODE_STEP && mode != MODE_STEP_PREDICT; }
#else
__host__ __device__ constexpr bool writes_out(int mode) { return mode != MODE_STEP; }
#endif

// ---- vector memory access -------------------------------------------------

template <int VEC>
struct Vec {
  float v[VEC];
};

// CACHE: 0 default, 1 streaming (.cs: evict-first in L1/L2, data touched once),
//        2 loads bypass L1 allocation (.L1::no_allocate), default stores.
template <int VEC, int CACHE, bool READ_ONLY>
__device__ __forceinline__ Vec<VEC> vload(const float* p) {
  Vec<VEC> r;
  if constexpr (VEC == 8) {
    if constexpr (CACHE == 1) {
      asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                     "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                   : "l"(p));
    } else if constexpr (CACHE == 2 && READ_ONLY) {
      asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                     "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                   : "l"(p));
    } else if constexpr (CACHE == 2) {
      asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                     "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                   : "l"(p));
    } else {
      asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                     "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                   : "l"(p));
    }
  } else if constexpr (VEC == 4) {
    if constexpr (CACHE == 1) {
      asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                   : "l"(p));
    } else if constexpr (CACHE == 2 && READ_ONLY) {
      asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                   : "l"(p));
    } else if constexpr (CACHE == 2) {
      asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                   : "l"(p));
    } else {
      asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                   : "l"(p));
    }
  } else {
    r.v[0] = CACHE == 1 ? __ldcs(p) : *p;
  }
  return r;
}

template <int VEC, int CACHE>
__device__ __forceinline__ void vstore(float* p, const Vec<VEC>& r) {
  if constexpr (VEC == 8) {
    if constexpr (CACHE == 1) {
      asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]),
                   "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]),
                   "f"(r.v[7])
                   : "memory");
    } else {
      asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]),
                   "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]),
                   "f"(r.v[7])
                   : "memory");
    }
  } else if constexpr (VEC == 4) {
    if constexpr (CACHE == 1) {
      asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]),
                   "f"(r.v[2]), "f"(r.v[3])
                   : "memory");
    } else {
      asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]),
                   "f"(r.v[2]), "f"(r.v[3])
                   : "memory");
    }
  } else {
    if (CACHE == 1)
      __stcs(p, r.v[0]);
    else
      *p = r.v[0];
  }
}

// CACHE 4 = "mixed": the weights and the predicted weights keep normal L2
// priority (the stage's next GEMMs read them right away — pipeline-sized
// stages fit in L2), the gradient and the optimizer state stream (.cs: not
// needed again until the next update). Per-stream policy for each CACHE:
enum Stream_ : int { S_W = 0, S_G = 1, S_STATE = 2, S_OUT = 3 };
__host__ __device__ constexpr int pol(int cache, int stream) {
  return cache == 4 ? ((stream == S_W || stream == S_OUT) ? 0 : 1) : cache;
}

template <int KIND, int MODE, int VEC, int CACHE>
__device__ __forceinline__ void do_vec(const Args& a, const Coef& c, int64_t vi, int64_t& bad) {
  const int64_t base = vi * VEC;
  Vec<VEC> w{}, g{}, s1{}, s2{}, out{};
  if constexpr (uses_w(MODE)) w = vload<VEC, pol(CACHE, S_W), !writes_w(MODE)>(a.w + base);
  if constexpr (uses_g(MODE)) g = vload<VEC, pol(CACHE, S_G), true>(a.g + base);
  if constexpr (uses_s1(MODE)) s1 = vload<VEC, pol(CACHE, S_STATE), !writes_state(MODE)>(a.s1 + base);
  if constexpr (uses_s2(KIND, MODE)) s2 = vload<VEC, pol(CACHE, S_STATE), !writes_state(MODE)>(a.s2 + base);
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    bool e = false;
    elem<KIND, MODE>(c, w.v[j], g.v[j], s1.v[j], s2.v[j], out.v[j], e);
    if (e && bad == INT64_MAX) bad = base + j;
  }
  if constexpr (writes_w(MODE)) vstore<VEC, pol(CACHE, S_W)>(a.w + base, w);
  if constexpr (writes_state(MODE)) {
    vstore<VEC, pol(CACHE, S_STATE)>(a.s1 + base, s1);
    if constexpr (KIND != PO_SGDM) vstore<VEC, pol(CACHE, S_STATE)>(a.s2 + base, s2);
  }
  if constexpr (writes_out(MODE)) vstore<VEC, pol(CACHE, S_OUT)>(a.out + base, out);
}

// UNROLL code for the software-pipelined loop (po_launch.unroll = 3)
constexpr int kPrefetch = 3;

// Persistent grid-stride stream. Each thread issues UNROLL independent vector
// loads per stream before the first use (memory-level parallelism: Little's law
// at ~6.5 TB/s x ~0.8 us needs ~5 MB in flight chip-wide, ~35 KB per SM).
template <int KIND, int MODE, int VEC, int CACHE, int UNROLL>
__global__ void __launch_bounds__(512) po_stream_kernel(const Args a) {
  pdl_wait();  // PDL launches: the predecessor's writes (gradient, coefficients) are complete
  pdl_trigger();
  const int64_t nv = a.n / VEC;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t bad = INT64_MAX;
  int64_t i = tid;
  const Coef c = load_coef(a);

  if constexpr (UNROLL == kPrefetch) {
    // Software pipeline: the next grid-stride vector's loads are issued before
    // this vector's arithmetic and stores, so one vector per stream stays in
    // flight while the (division + square-root) math of the current one runs.
    // The elements a thread touches are its own (disjoint grid-stride
    // partition), so hoisting the next loads above the current stores is safe.
    Vec<VEC> w{}, g{}, s1{}, s2{};
    auto load = [&](int64_t vi, Vec<VEC>& w_, Vec<VEC>& g_, Vec<VEC>& s1_, Vec<VEC>& s2_) {
      const int64_t base = vi * VEC;
      if constexpr (uses_w(MODE)) w_ = vload<VEC, pol(CACHE, S_W), !writes_w(MODE)>(a.w + base);
      if constexpr (uses_g(MODE)) g_ = vload<VEC, pol(CACHE, S_G), true>(a.g + base);
      if constexpr (uses_s1(MODE)) s1_ = vload<VEC, pol(CACHE, S_STATE), !writes_state(MODE)>(a.s1 + base);
      if constexpr (uses_s2(KIND, MODE)) s2_ = vload<VEC, pol(CACHE, S_STATE), !writes_state(MODE)>(a.s2 + base);
    };
    if (i < nv) load(i, w, g, s1, s2);
    for (; i < nv; i += stride) {
      const int64_t base = i * VEC;
      Vec<VEC> nw{}, ng{}, ns1{}, ns2{}, out;
      if (i + stride < nv) load(i + stride, nw, ng, ns1, ns2);
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        bool e = false;
        elem<KIND, MODE>(c, w.v[j], g.v[j], s1.v[j], s2.v[j], out.v[j], e);
        if (e && bad == INT64_MAX) bad = base + j;
      }
      if constexpr (writes_w(MODE)) vstore<VEC, pol(CACHE, S_W)>(a.w + base, w);
      if constexpr (writes_state(MODE)) {
        vstore<VEC, pol(CACHE, S_STATE)>(a.s1 + base, s1);
        if constexpr (KIND != PO_SGDM) vstore<VEC, pol(CACHE, S_STATE)>(a.s2 + base, s2);
      }
      if constexpr (writes_out(MODE)) vstore<VEC, pol(CACHE, S_OUT)>(a.out + base, out);
      w = nw;
      g = ng;
      s1 = ns1;
      s2 = ns2;
    }
  }

  for (; UNROLL != kPrefetch && i + (UNROLL - 1) * stride < nv; i += UNROLL * stride) {
    constexpr int U = UNROLL == kPrefetch ? 1 : UNROLL;
    Vec<VEC> w[U], g[U], s1[U], s2[U], out[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t base = (i + u * stride) * VEC;
      if constexpr (uses_w(MODE)) w[u] = vload<VEC, pol(CACHE, S_W), !writes_w(MODE)>(a.w + base);
      if constexpr (uses_g(MODE)) g[u] = vload<VEC, pol(CACHE, S_G), true>(a.g + base);
      if constexpr (uses_s1(MODE)) s1[u] = vload<VEC, pol(CACHE, S_STATE), !writes_state(MODE)>(a.s1 + base);
      if constexpr (uses_s2(KIND, MODE)) s2[u] = vload<VEC, pol(CACHE, S_STATE), !writes_state(MODE)>(a.s2 + base);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t base = (i + u * stride) * VEC;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        bool e = false;
        elem<KIND, MODE>(c, w[u].v[j], g[u].v[j], s1[u].v[j], s2[u].v[j], out[u].v[j], e);
        if (e && bad == INT64_MAX) bad = base + j;
      }
      if constexpr (writes_w(MODE)) vstore<VEC, pol(CACHE, S_W)>(a.w + base, w[u]);
      if constexpr (writes_state(MODE)) {
        vstore<VEC, pol(CACHE, S_STATE)>(a.s1 + base, s1[u]);
        if constexpr (KIND != PO_SGDM) vstore<VEC, pol(CACHE, S_STATE)>(a.s2 + base, s2[u]);
      }
      if constexpr (writes_out(MODE)) vstore<VEC, pol(CACHE, S_OUT)>(a.out + base, out[u]);
    }
  }
  for (; i < nv; i += stride) do_vec<KIND, MODE, VEC, CACHE>(a, c, i, bad);

  // scalar tail [nv*VEC, n): fewer than VEC elements
  const int64_t t = nv * VEC + tid;
  if (t < a.n) {
    float w = 0.f, g = 0.f, s1 = 0.f, s2 = 0.f, out = 0.f;
    if constexpr (uses_w(MODE)) w = a.w[t];
    if constexpr (uses_g(MODE)) g = a.g[t];
    if constexpr (uses_s1(MODE)) s1 = a.s1[t];
    if constexpr (uses_s2(KIND, MODE)) s2 = a.s2[t];
    bool e = false;
    elem<KIND, MODE>(c, w, g, s1, s2, out, e);
    if (e && bad == INT64_MAX) bad = t;
    if constexpr (writes_w(MODE)) a.w[t] = w;
    if constexpr (writes_state(MODE)) {
      a.s1[t] = s1;
      if constexpr (KIND != PO_SGDM) a.s2[t] = s2;
    }
    if constexpr (writes_out(MODE)) a.out[t] = out;
  }
  if (a.bad != nullptr && bad != INT64_MAX) atomicMin(a.bad, (unsigned long long)bad);
}

// ---- host side ---------------------------------------------------------------

constexpr int kMaxDevices = 64;
int g_sm_count[kMaxDevices] = {0};

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= kMaxDevices) return 148;
  if (g_sm_count[dev] == 0) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
    g_sm_count[dev] = sms;
  }
  return g_sm_count[dev];
}

bool aligned(const void* p, int bytes) {
  return p == nullptr || (reinterpret_cast<uintptr_t>(p) % (uintptr_t)bytes) == 0;
}

// Only the hot modes (K1/K2/K3) get every launch-shape variant; the
// reference-compatibility reads use the default shape.
__host__ __device__ constexpr bool tunable(int mode) {
  return mode == MODE_STEP || mode == MODE_PREDICT || mode == MODE_STEP_PREDICT;
}

struct Shape {
  int vec, cache, unroll;
};

template <int KIND, int MODE, int VEC, int CACHE>
cudaError_t launch_unroll(const Args& a, const Shape& sh, dim3 grid, dim3 block, cudaStream_t s) {
  if constexpr (tunable(MODE) && VEC > 1) {
    switch (sh.unroll) {
      case 1: pdl_launch(po_stream_kernel<KIND, MODE, VEC, CACHE, 1>, grid, block, 0, s, a); break;
      case kPrefetch: pdl_launch(po_stream_kernel<KIND, MODE, VEC, CACHE, kPrefetch>, grid, block, 0, s, a); break;
      case 4: pdl_launch(po_stream_kernel<KIND, MODE, VEC, CACHE, 4>, grid, block, 0, s, a); break;
      default: pdl_launch(po_stream_kernel<KIND, MODE, VEC, CACHE, 2>, grid, block, 0, s, a); break;
    }
  } else {
    pdl_launch(po_stream_kernel<KIND, MODE, VEC, CACHE, (VEC > 1 ? 2 : 4)>, grid, block, 0, s, a);
  }
  return cudaGetLastError();
}

template <int KIND, int MODE, int VEC>
cudaError_t launch_cache(const Args& a, const Shape& sh, dim3 grid, dim3 block, cudaStream_t s) {
  if constexpr (tunable(MODE) && VEC > 1) {
    switch (sh.cache) {
      case 0: return launch_unroll<KIND, MODE, VEC, 0>(a, sh, grid, block, s);
      case 2: return launch_unroll<KIND, MODE, VEC, 2>(a, sh, grid, block, s);
      case 4: return launch_unroll<KIND, MODE, VEC, 4>(a, sh, grid, block, s);
      default: return launch_unroll<KIND, MODE, VEC, 1>(a, sh, grid, block, s);
    }
  } else {
    return launch_unroll<KIND, MODE, VEC, 1>(a, sh, grid, block, s);
  }
}

template <int KIND, int MODE>
cudaError_t launch_vec(const Args& a, const Shape& sh, dim3 grid, dim3 block, cudaStream_t s) {
  switch (sh.vec) {
    case 8: return launch_cache<KIND, MODE, 8>(a, sh, grid, block, s);
    case 4: return launch_cache<KIND, MODE, 4>(a, sh, grid, block, s);
    default: return launch_cache<KIND, MODE, 1>(a, sh, grid, block, s);
  }
}

template <int MODE>
cudaError_t launch_kind(int kind, const Args& a, const Shape& sh, dim3 grid, dim3 block,
                        cudaStream_t s) {
  switch (kind) {
    case PO_SGDM: return launch_vec<PO_SGDM, MODE>(a, sh, grid, block, s);
    case PO_ADAM: return launch_vec<PO_ADAM, MODE>(a, sh, grid, block, s);
    default: return launch_vec<PO_ADAMW, MODE>(a, sh, grid, block, s);
  }
}

cudaError_t dispatch(int kind, int mode, const Args& a, const Shape& sh, dim3 grid, dim3 block,
                     cudaStream_t s) {
  switch (mode) {
    case MODE_STEP: return launch_kind<MODE_STEP>(kind, a, sh, grid, block, s);
    case MODE_STEP_DIR: return launch_kind<MODE_STEP_DIR>(kind, a, sh, grid, block, s);
    case MODE_PREDICT: return launch_kind<MODE_PREDICT>(kind, a, sh, grid, block, s);
    case MODE_PREDICT_ZERO: return launch_vec<PO_SGDM, MODE_PREDICT_ZERO>(a, sh, grid, block, s);
    case MODE_STEP_PREDICT: return launch_kind<MODE_STEP_PREDICT>(kind, a, sh, grid, block, s);
    case MODE_DIRECTION: return launch_kind<MODE_DIRECTION>(kind, a, sh, grid, block, s);
    case MODE_DIRECTION_ZERO:
      return launch_vec<PO_SGDM, MODE_DIRECTION_ZERO>(a, sh, grid, block, s);
    default: return launch_vec<PO_SGDM, MODE_AXPY>(a, sh, grid, block, s);
  }
}

// Default launch shapes per (mode, kind), from the 2^30-element B200 sweep
// (scripts/kernel_sweep.py --tune-all; profiles/r1_kernel_tune.md): all use
// 256-bit vectors; `unroll` vectors per stream in flight per thread.
struct DefaultShape {
  int block, ctas_per_sm, unroll, cache;
};

DefaultShape default_shape(int kind, int mode, int64_t n) {
  const bool sg = kind == PO_SGDM;
  // pipeline-stage sizes (< 32 M elements, the 1F1B configs' 0.01-20 M-param
  // stages): many small CTAs (pipeline stages run concurrently with other
  // stages' kernels, profiles/r1_pipeline.md), streaming stores, and a full
  // SM (16 x 128 threads) with one vector per stream each — the best or tied
  // shape for K1 and K3 (SGDM and Adam) at 2^20 / 2^22 / 2^24 in the L2-flushed
  // round-2 sweep (profiles/r2_kernel_tune_small.jsonl): K1 Adam at 2^24
  // 53.3 -> 45.1 us (0.77 -> 0.91 of copy), at 2^22 20.5 -> 16.4 us
  // (the prefetching loop is faster for K3 Adam alone at 2^24, 6,362 ->
  // 6,518 GB/s L2-flushed, profiles/r2_ab_small.jsonl, but costs config 1's
  // 1F1B run 3 % with prediction on, where K3 shares the GPU with the other
  // stages' GEMMs: not adopted)
  if (n < (int64_t(1) << 25)) return DefaultShape{128, 16, 1, 1};
  // >= 2^25: re-tuned at 1e9 with the one-division Adam direction
  // (profiles/r2_tune_1e9.jsonl, all shapes timed in alternation on one box):
  // K3 Adam 320 threads x 1 CTA/SM with the next vector prefetched 6,543 GB/s
  // (512 x 1, one vector in flight: 6,244); K2 Adam 512 x 1, one vector in
  // flight 6,623 (512 x 1 x 2 plain: 6,228). More requests in flight than
  // these is slower: the DRAM sees finer read/write interleaving.
  switch (mode) {
    case MODE_PREDICT: return sg ? DefaultShape{256, 8, 2, 1} : DefaultShape{512, 2, 1, 1};
    case MODE_STEP: return sg ? DefaultShape{512, 1, 1, 1} : DefaultShape{512, 1, 1, 1};
    case MODE_STEP_PREDICT:
      if (sg) return DefaultShape{384, 1, 1, 1};
      return DefaultShape{320, 1, 3, 1};  // Adam and AdamW
    default: return DefaultShape{256, 4, 2, 1};
  }
}
constexpr int kDefaultVec = 8;

int run(int kind, int mode, Args a, const po_launch* L, cudaStream_t s) {
  if (a.n < 0) return PO_EINVAL;
  if (a.n == 0) return 0;
  const DefaultShape d = default_shape(kind, mode, a.n);
  int block = (L && L->block > 0) ? L->block : d.block;
  int cps = (L && L->ctas_per_sm > 0) ? L->ctas_per_sm : d.ctas_per_sm;
  int vec = (L && L->vec > 0) ? L->vec : kDefaultVec;
  int cache = (L && L->cache > 0 && L->cache <= 4) ? L->cache : d.cache;
  if (L && L->cache == 3) cache = 0;  // explicit plain ld/st request
  int unroll = (L && L->unroll > 0) ? L->unroll : d.unroll;
  // W_hat written over the gradient (the runtime's staging-in-gradient): no
  // non-coherent (.nc) gradient loads on memory this launch writes
  if (cache == 2 && a.out != nullptr && a.out == a.g) cache = 1;
  if (block % 32 != 0 || block > 512) return PO_EINVAL;
  if (unroll != 1 && unroll != 2 && unroll != 4 && unroll != kPrefetch) return PO_EINVAL;
  if (vec != 8 && vec != 4 && vec != 1) return PO_EINVAL;
  // fall back to narrower vectors when any stream is misaligned
  const void* ptrs[5] = {a.w, a.g, a.s1, a.s2, a.out};
  while (vec > 1) {
    bool ok = true;
    for (const void* p : ptrs) ok = ok && aligned(p, vec * 4);
    if (ok) break;
    vec = vec == 8 ? 4 : 1;
  }
  const int64_t nv = a.n / vec;
  const int64_t tail = a.n - nv * vec;
  int64_t want = (nv + block - 1) / block;
  if (want < 1) want = 1;
  const int64_t tail_blocks = (tail + block - 1) / block;
  if (want < tail_blocks) want = tail_blocks;
  int64_t cap = (int64_t)sm_count() * cps;
  int64_t grid = want < cap ? want : cap;
  const Shape sh{vec, cache, unroll};
  cudaError_t e = dispatch(kind, mode, a, sh, dim3((unsigned)grid), dim3(block), s);
  return e == cudaSuccess ? 0 : (int)e;
}

bool valid_hp(const po_hparams* hp) {
  if (hp == nullptr) return false;
  if (hp->kind != PO_SGDM && hp->kind != PO_ADAM && hp->kind != PO_ADAMW) return false;
  return true;
}

// ---- hybrid DP x PP: gradient reduction over peer memory fused into K3 -------
//
// Each data-parallel replica of a stage owns a flat gradient buffer; the
// replicas map each other's buffers (CUDA IPC over NVLink / NVSwitch). The
// fused kernel reads the dp gradients of every element straight from peer
// memory, sums them in RANK ORDER (so every replica computes the identical
// mean and the replicas stay bit-identical), and applies K3 in the same pass:
// no reduced gradient is written to HBM and read back, no separate collective
// launch. A replica signals "my gradient of epoch e is complete" with one
// release store per peer into the peer's flag array (po_dp_signal, enqueued
// after its backward); a one-CTA kernel acquire-waits on the local flags
// before the streaming kernel touches any peer gradient. Gradients are double-buffered by
// epoch parity, which makes a second "consumed" handshake unnecessary: a
// replica overwrites parity p again only in epoch e+2, after it observed every
// peer's epoch-(e+1) signal, which each peer issued after its epoch-e update
// (stream order) had finished reading.

constexpr int kMaxDp = 8;

struct DpArgs {
  Args a;                             // w, s1, s2, out (w_hat), n, bad, coefficients
  const float* grads[kMaxDp];         // every replica's gradient (this epoch's parity), rank order
  int dp;
  float inv_dp;
  const long long* flags;             // local [dp]: last epoch each replica signalled
  long long epoch;
  long long timeout_cycles;
  int* status;                        // set to 1 if a peer never signalled (kernel then skips)
};

__device__ __forceinline__ long long ld_acquire_sys(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One 32-thread CTA acquire-waits for every replica's signal. It runs BEFORE
// the streaming kernel (stream order) so the wait occupies one CTA, never the
// whole GPU: NCCL kernels of the pipeline exchanges keep running beside it
// (a full-grid spin could starve them and close a dependency cycle across
// replicas).
__global__ void po_dp_wait_kernel(const long long* flags, int dp, long long epoch, long long timeout_cycles,
                                  int* status, const long long* epoch_dev) {
  if (threadIdx.x != 0) return;
  if (*(volatile int*)status != 0) return;  // already failed: do not wait again
  if (epoch_dev != nullptr) epoch = *(volatile const long long*)epoch_dev;  // graph replays: device counter
  const long long t0 = clock64();
  for (int r = 0; r < dp; ++r) {
    while (ld_acquire_sys(flags + r) < epoch) {
      if (clock64() - t0 > timeout_cycles) {
        atomicExch(status, 1);
        return;
      }
      __nanosleep(512);
    }
  }
}

// DP is a template parameter so every replica's gradient load of an element
// is issued before the first add (dp independent NVLink/HBM loads in flight
// per vector, plus W and the state), then summed in rank order.
template <int KIND, int VEC, int DP>
__global__ void __launch_bounds__(512) po_dp_kernel(const DpArgs d) {
  if (*(volatile int*)d.status != 0) return;  // a replica never signalled: update nothing
  const Args& a = d.a;
  const Coef c = load_coef(a);
  const int64_t nv = a.n / VEC;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t bad = INT64_MAX;
  // PF (dp <= 2): the software-pipelined loop of K3 — the next vector's
  // loads (dp gradients, W, state) issued before this vector's arithmetic
  constexpr bool PF = DP <= 2;
  Vec<VEC> gr[DP], w{}, s1{}, s2{};
  auto load = [&](int64_t base, Vec<VEC>(&gr_)[DP], Vec<VEC>& w_, Vec<VEC>& s1_, Vec<VEC>& s2_) {
#pragma unroll
    for (int r = 0; r < DP; ++r) gr_[r] = vload<VEC, 1, true>(d.grads[r] + base);
    w_ = vload<VEC, 1, false>(a.w + base);
    s1_ = vload<VEC, 1, false>(a.s1 + base);
    if constexpr (KIND != PO_SGDM) s2_ = vload<VEC, 1, false>(a.s2 + base);
  };
  if (PF && tid < nv) load(tid * VEC, gr, w, s1, s2);
  for (int64_t i = tid; i < nv; i += stride) {
    const int64_t base = i * VEC;
    Vec<VEC> ngr[PF ? DP : 1], nw{}, ns1{}, ns2{};
    if constexpr (PF) {
      if (i + stride < nv) load((i + stride) * VEC, ngr, nw, ns1, ns2);
    } else {
      load(base, gr, w, s1, s2);
    }
    Vec<VEC> out;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float g = gr[0].v[j];
#pragma unroll
      for (int r = 1; r < DP; ++r) g = __fadd_rn(g, gr[r].v[j]);  // rank order
      bool e = false;
      elem<KIND, MODE_STEP_PREDICT>(c, w.v[j], DP == 1 ? g : __fmul_rn(g, d.inv_dp), s1.v[j], s2.v[j], out.v[j], e);
      if (e && bad == INT64_MAX) bad = base + j;
    }
    vstore<VEC, 1>(a.w + base, w);
    vstore<VEC, 1>(a.s1 + base, s1);
    if constexpr (KIND != PO_SGDM) vstore<VEC, 1>(a.s2 + base, s2);
    vstore<VEC, 1>(a.out + base, out);
    if constexpr (PF) {
#pragma unroll
      for (int r = 0; r < DP; ++r) gr[r] = ngr[r];
      w = nw;
      s1 = ns1;
      s2 = ns2;
    }
  }
  const int64_t t = nv * VEC + tid;  // scalar tail
  if (t < a.n) {
    float g = d.grads[0][t];
#pragma unroll
    for (int r = 1; r < DP; ++r) g = __fadd_rn(g, d.grads[r][t]);
    float w = a.w[t], s1 = a.s1[t], s2 = (KIND != PO_SGDM) ? a.s2[t] : 0.f, out = 0.f;
    bool e = false;
    elem<KIND, MODE_STEP_PREDICT>(c, w, DP == 1 ? g : __fmul_rn(g, d.inv_dp), s1, s2, out, e);
    if (e && bad == INT64_MAX) bad = t;
    a.w[t] = w;
    a.s1[t] = s1;
    if constexpr (KIND != PO_SGDM) a.s2[t] = s2;
    a.out[t] = out;
  }
  if (a.bad != nullptr && bad != INT64_MAX) atomicMin(a.bad, (unsigned long long)bad);
}

__global__ void po_dp_signal_kernel(long long* const* slots, int dp, long long epoch, long long* epoch_ctr) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (epoch_ctr != nullptr) {  // device-side epoch: advanced here, read by the wait kernel
      epoch = *(volatile long long*)epoch_ctr + 1;
      *epoch_ctr = epoch;
    }
    __threadfence_system();
    for (int r = 0; r < dp; ++r)
      asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(slots[r]), "l"(epoch) : "memory");
  }
}

// ---- hybrid DP x PP, sharded: reduce-scatter + K3 + all-gather in ONE pass ----
//
// Replica `rank` owns the contiguous shard [lo, hi) of the stage's flat
// buffers. For each of its elements it sums the dp replicas' gradients (rank
// order over peer memory, or multimem.ld_reduce through the NVSwitch when a
// multicast mapping is given), applies K3 against its own copy of W / state,
// and writes W', m', v' and W_hat into EVERY replica's buffers (dp peer
// stores, or one multimem.st). Each element is computed exactly once, so the
// replicas stay bit-identical whatever the reduction order; per GPU the HBM
// traffic is ~(20 + 12/dp) B/param instead of (28 + 4 dp) B/param for
// po_step_predict_dp (every replica reading every gradient). A done-barrier
// (po_dp_done_kernel + a wait) follows: a replica's next forward reads W_hat
// written by all owners.

struct DpShardArgs {
  Args a;                              // coefficients (c or dc), n = whole stage
  float* w[kMaxDp];                    // every replica's buffers, rank order
  float* s1[kMaxDp];
  float* s2[kMaxDp];
  float* out[kMaxDp];                  // W_hat (all null: plain step)
  const float* grads[kMaxDp];
  unsigned long long* bad[kMaxDp];     // every replica's non-finite flag (nullable)
  float* mc_g;                         // multicast (NVLS) addresses, all null = peer stores
  float* mc_w;
  float* mc_s1;
  float* mc_s2;
  float* mc_out;
  int dp, rank;
  int64_t lo, hi;
  float inv_dp;
  int* status;
};

template <int VEC>
__device__ __forceinline__ Vec<VEC> mc_ld_reduce(const float* p) {
  Vec<VEC> r;
  if constexpr (VEC == 1) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r.v[0]) : "l"(p) : "memory");
  } else {
#pragma unroll
    for (int h = 0; h < VEC; h += 4)
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(r.v[h]), "=f"(r.v[h + 1]), "=f"(r.v[h + 2]), "=f"(r.v[h + 3])
                   : "l"(p + h)
                   : "memory");
  }
  return r;
}

template <int VEC>
__device__ __forceinline__ void mc_store(float* p, const Vec<VEC>& r) {
  if constexpr (VEC == 1) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(r.v[0]) : "memory");
  } else {
#pragma unroll
    for (int h = 0; h < VEC; h += 4)
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + h), "f"(r.v[h]),
                   "f"(r.v[h + 1]), "f"(r.v[h + 2]), "f"(r.v[h + 3])
                   : "memory");
  }
}

template <int KIND, int VEC, int DP, bool MC>
__device__ __forceinline__ void shard_vec(const DpShardArgs& d, const Coef& c, int64_t base, int64_t& bad) {
  Vec<VEC> g;
  if constexpr (MC) {
    g = mc_ld_reduce<VEC>(d.mc_g + base);
  } else {
    Vec<VEC> gr[DP];
#pragma unroll
    for (int r = 0; r < DP; ++r) gr[r] = vload<VEC, 1, true>(d.grads[r] + base);
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float x = gr[0].v[j];
#pragma unroll
      for (int r = 1; r < DP; ++r) x = __fadd_rn(x, gr[r].v[j]);  // rank order
      g.v[j] = x;
    }
  }
  Vec<VEC> w = vload<VEC, 1, false>(d.w[d.rank] + base);
  Vec<VEC> s1 = vload<VEC, 1, false>(d.s1[d.rank] + base);
  Vec<VEC> s2{};
  if constexpr (KIND != PO_SGDM) s2 = vload<VEC, 1, false>(d.s2[d.rank] + base);
  Vec<VEC> out;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    bool e = false;
    elem<KIND, MODE_STEP_PREDICT>(c, w.v[j], DP == 1 ? g.v[j] : __fmul_rn(g.v[j], d.inv_dp), s1.v[j], s2.v[j],
                                  out.v[j], e);
    if (e && bad == INT64_MAX) bad = base + j;
  }
  const bool write_out = MC ? d.mc_out != nullptr : d.out[0] != nullptr;
  if constexpr (MC) {
    mc_store<VEC>(d.mc_w + base, w);
    mc_store<VEC>(d.mc_s1 + base, s1);
    if constexpr (KIND != PO_SGDM) mc_store<VEC>(d.mc_s2 + base, s2);
    if (write_out) mc_store<VEC>(d.mc_out + base, out);
  } else {
    // own copy first (streaming stores, as K3), then the peers (plain stores)
    vstore<VEC, 1>(d.w[d.rank] + base, w);
    vstore<VEC, 1>(d.s1[d.rank] + base, s1);
    if constexpr (KIND != PO_SGDM) vstore<VEC, 1>(d.s2[d.rank] + base, s2);
    if (write_out) vstore<VEC, 1>(d.out[d.rank] + base, out);
#pragma unroll
    for (int q = 1; q < DP; ++q) {
      const int r = (d.rank + q) % DP;
      vstore<VEC, 0>(d.w[r] + base, w);
      vstore<VEC, 0>(d.s1[r] + base, s1);
      if constexpr (KIND != PO_SGDM) vstore<VEC, 0>(d.s2[r] + base, s2);
      if (write_out) vstore<VEC, 0>(d.out[r] + base, out);
    }
  }
}

template <int KIND, int VEC, int DP, bool MC>
__global__ void __launch_bounds__(512) po_dp_shard_kernel(const DpShardArgs d) {
  if (*(volatile int*)d.status != 0) return;  // a replica never signalled: update nothing
  const Coef c = load_coef(d.a);
  const int64_t nv = (d.hi - d.lo) / VEC;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t bad = INT64_MAX;
  for (int64_t i = tid; i < nv; i += stride) shard_vec<KIND, VEC, DP, MC>(d, c, d.lo + i * VEC, bad);
  const int64_t t = d.lo + nv * VEC + tid;  // scalar tail of the last shard
  if (t < d.hi) shard_vec<KIND, 1, DP, MC>(d, c, t, bad);
  if (bad != INT64_MAX)
    for (int r = 0; r < DP; ++r)
      if (d.bad[r] != nullptr) atomicMin(d.bad[r], (unsigned long long)bad);
}

// After the shard kernel (stream order): release-store the epoch into this
// replica's slot of every replica's done array. Skipped when the gradient
// wait timed out, so the peers time out too instead of reading a half update.
__global__ void po_dp_done_kernel(long long* const* slots, int dp, long long epoch, const long long* epoch_dev,
                                  const int* status) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (*(volatile const int*)status != 0) return;
    if (epoch_dev != nullptr) epoch = *(volatile const long long*)epoch_dev;
    __threadfence_system();
    for (int r = 0; r < dp; ++r)
      asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(slots[r]), "l"(epoch) : "memory");
  }
}

template <int KIND, int VEC, bool MC>
cudaError_t launch_shard_vec(const DpShardArgs& d, dim3 grid, dim3 block, cudaStream_t s) {
  switch (d.dp) {
    case 1: po_dp_shard_kernel<KIND, VEC, 1, MC><<<grid, block, 0, s>>>(d); break;
    case 2: po_dp_shard_kernel<KIND, VEC, 2, MC><<<grid, block, 0, s>>>(d); break;
    case 3: po_dp_shard_kernel<KIND, VEC, 3, MC><<<grid, block, 0, s>>>(d); break;
    case 4: po_dp_shard_kernel<KIND, VEC, 4, MC><<<grid, block, 0, s>>>(d); break;
    case 5: po_dp_shard_kernel<KIND, VEC, 5, MC><<<grid, block, 0, s>>>(d); break;
    case 6: po_dp_shard_kernel<KIND, VEC, 6, MC><<<grid, block, 0, s>>>(d); break;
    case 7: po_dp_shard_kernel<KIND, VEC, 7, MC><<<grid, block, 0, s>>>(d); break;
    default: po_dp_shard_kernel<KIND, VEC, 8, MC><<<grid, block, 0, s>>>(d); break;
  }
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_shard(const DpShardArgs& d, int vec, bool mc, dim3 grid, dim3 block, cudaStream_t s) {
  if (mc) {
    if (vec == 8) return launch_shard_vec<KIND, 8, true>(d, grid, block, s);
    if (vec == 4) return launch_shard_vec<KIND, 4, true>(d, grid, block, s);
    return launch_shard_vec<KIND, 1, true>(d, grid, block, s);
  }
  if (vec == 8) return launch_shard_vec<KIND, 8, false>(d, grid, block, s);
  if (vec == 4) return launch_shard_vec<KIND, 4, false>(d, grid, block, s);
  return launch_shard_vec<KIND, 1, false>(d, grid, block, s);
}

template <int KIND, int VEC>
cudaError_t launch_dp_vec(const DpArgs& d, dim3 grid, dim3 block, cudaStream_t s) {
  switch (d.dp) {
    case 1: po_dp_kernel<KIND, VEC, 1><<<grid, block, 0, s>>>(d); break;
    case 2: po_dp_kernel<KIND, VEC, 2><<<grid, block, 0, s>>>(d); break;
    case 3: po_dp_kernel<KIND, VEC, 3><<<grid, block, 0, s>>>(d); break;
    case 4: po_dp_kernel<KIND, VEC, 4><<<grid, block, 0, s>>>(d); break;
    case 5: po_dp_kernel<KIND, VEC, 5><<<grid, block, 0, s>>>(d); break;
    case 6: po_dp_kernel<KIND, VEC, 6><<<grid, block, 0, s>>>(d); break;
    case 7: po_dp_kernel<KIND, VEC, 7><<<grid, block, 0, s>>>(d); break;
    default: po_dp_kernel<KIND, VEC, 8><<<grid, block, 0, s>>>(d); break;
  }
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_dp(const DpArgs& d, int vec, dim3 grid, dim3 block, cudaStream_t s) {
  if (vec == 8) return launch_dp_vec<KIND, 8>(d, grid, block, s);
  if (vec == 4) return launch_dp_vec<KIND, 4>(d, grid, block, s);
  return launch_dp_vec<KIND, 1>(d, grid, block, s);
}

}  // namespace

extern "C" {

static int32_t g_pdl = 0;
int po_set_pdl(int32_t on) {
  g_pdl = on ? 1 : 0;
  return 0;
}
int po_get_pdl(void) { return g_pdl; }

int po_abi_version(void) { return PO_ABI_VERSION; }

const char* po_strerror(int code) {
  if (code == 0) return "ok";
  if (code == PO_EINVAL) return "invalid argument";
  if (code >= PO_EDRIVER_BASE) {  // resolved at run time: no link-time libcuda dependency
    using Fn = CUresult (*)(CUresult, const char**);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    const char* s = nullptr;
    if (cudaGetDriverEntryPoint("cuGetErrorString", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      reinterpret_cast<Fn>(fn)((CUresult)(code - PO_EDRIVER_BASE), &s);
    return s != nullptr ? s : "CUDA driver error";
  }
  return cudaGetErrorString((cudaError_t)code);
}

int po_version_difference(int64_t depth, int64_t rank, int64_t* out) {
  // optim.py:158-167
  if (out == nullptr || depth < 1 || rank < 0 || rank >= depth) return PO_EINVAL;
  *out = depth - rank - 1;
  return 0;
}

int po_step(const po_hparams* hp, float* w, const float* g, float* state1, float* state2,
            float* dir_out, int64_t n, double lr, int64_t step_count, int64_t* nonfinite_index,
            const po_launch* launch, void* stream) {
  if (!valid_hp(hp) || step_count < 0) return PO_EINVAL;
  if (n > 0 && (w == nullptr || g == nullptr || state1 == nullptr)) return PO_EINVAL;
  if (n > 0 && hp->kind != PO_SGDM && state2 == nullptr) return PO_EINVAL;
  Args a{w, g, state1, hp->kind == PO_SGDM ? nullptr : state2, dir_out, n,
         reinterpret_cast<unsigned long long*>(nonfinite_index), nullptr,
         coef(hp, lr, 0.0, step_count + 1)};
  return run(hp->kind, dir_out ? MODE_STEP_DIR : MODE_STEP, a, launch, (cudaStream_t)stream);
}

int po_predict(const po_hparams* hp, const float* w, const float* state1, const float* state2,
               float* w_hat, int64_t n, double lr_times_s, int64_t step_count,
               const po_launch* launch, void* stream) {
  if (!valid_hp(hp) || step_count < 0) return PO_EINVAL;
  if (n > 0 && (w == nullptr || w_hat == nullptr)) return PO_EINVAL;
  const bool zero = step_count == 0;
  if (!zero && n > 0 && (state1 == nullptr || (hp->kind != PO_SGDM && state2 == nullptr)))
    return PO_EINVAL;
  Args a{const_cast<float*>(w), nullptr,
         zero ? nullptr : const_cast<float*>(state1),
         (zero || hp->kind == PO_SGDM) ? nullptr : const_cast<float*>(state2), w_hat, n, nullptr, nullptr,
         coef(hp, 0.0, lr_times_s, step_count)};
  return run(hp->kind, zero ? MODE_PREDICT_ZERO : MODE_PREDICT, a, launch, (cudaStream_t)stream);
}

int po_step_predict(const po_hparams* hp, float* w, const float* g, float* state1, float* state2,
                    float* w_hat, int64_t n, double lr, double lr_pred_times_s, int64_t step_count,
                    int64_t* nonfinite_index, const po_launch* launch, void* stream) {
  if (!valid_hp(hp) || step_count < 0) return PO_EINVAL;
  if (n > 0 && (w == nullptr || g == nullptr || state1 == nullptr || w_hat == nullptr))
    return PO_EINVAL;
  if (n > 0 && hp->kind != PO_SGDM && state2 == nullptr) return PO_EINVAL;
  Args a{w, g, state1, hp->kind == PO_SGDM ? nullptr : state2, w_hat, n,
         reinterpret_cast<unsigned long long*>(nonfinite_index), nullptr,
         coef(hp, lr, lr_pred_times_s, step_count + 1)};
  return run(hp->kind, MODE_STEP_PREDICT, a, launch, (cudaStream_t)stream);
}

int po_direction(const po_hparams* hp, const float* state1, const float* state2, float* dir_out,
                 int64_t n, int64_t step_count, const po_launch* launch, void* stream) {
  if (!valid_hp(hp) || step_count < 0) return PO_EINVAL;
  if (n > 0 && dir_out == nullptr) return PO_EINVAL;
  const bool zero = step_count == 0;
  if (!zero && n > 0 && (state1 == nullptr || (hp->kind != PO_SGDM && state2 == nullptr)))
    return PO_EINVAL;
  Args a{nullptr, nullptr, zero ? nullptr : const_cast<float*>(state1),
         (zero || hp->kind == PO_SGDM) ? nullptr : const_cast<float*>(state2), dir_out, n, nullptr, nullptr,
         coef(hp, 0.0, 0.0, step_count)};
  return run(hp->kind, zero ? MODE_DIRECTION_ZERO : MODE_DIRECTION, a, launch,
             (cudaStream_t)stream);
}

int po_axpy_predict(const float* w, const float* d, float* w_hat, int64_t n, double lr_times_s,
                    const po_launch* launch, void* stream) {
  if (n > 0 && (w == nullptr || d == nullptr || w_hat == nullptr)) return PO_EINVAL;
  Coef c;
  memset(&c, 0, sizeof(c));
  c.c_pred = (float)lr_times_s;
  Args a{const_cast<float*>(w), nullptr, const_cast<float*>(d), nullptr, w_hat, n, nullptr, nullptr, c};
  return run(PO_SGDM, MODE_AXPY, a, launch, (cudaStream_t)stream);
}

int po_coef_fill(const po_hparams* hp, int32_t which, double lr, double lr_times_s, int64_t step_count,
                 po_coef* out) {
  if (!valid_hp(hp) || out == nullptr || step_count < 0) return PO_EINVAL;
  Coef c;
  switch (which) {
    case PO_COEF_STEP: c = coef(hp, lr, 0.0, step_count + 1); break;
    case PO_COEF_PREDICT: c = coef(hp, 0.0, lr_times_s, step_count); break;  // t = 0 -> bc = 1
    case PO_COEF_STEP_PREDICT: c = coef(hp, lr, lr_times_s, step_count + 1); break;
    default: return PO_EINVAL;
  }
  out->lr = c.lr;
  out->c_pred = c.c_pred;
  out->inv_bc1 = c.ibc1;
  out->inv_bc2 = c.ibc2;
  return 0;
}

int po_step_dc(const po_hparams* hp, float* w, const float* g, float* state1, float* state2, int64_t n,
               const po_coef* coef_dev, int64_t* nonfinite_index, const po_launch* launch, void* stream) {
  if (!valid_hp(hp) || coef_dev == nullptr) return PO_EINVAL;
  if (n > 0 && (w == nullptr || g == nullptr || state1 == nullptr)) return PO_EINVAL;
  if (n > 0 && hp->kind != PO_SGDM && state2 == nullptr) return PO_EINVAL;
  Args a{w, g, state1, hp->kind == PO_SGDM ? nullptr : state2, nullptr, n,
         reinterpret_cast<unsigned long long*>(nonfinite_index), coef_dev, coef(hp, 0.0, 0.0, 1)};
  return run(hp->kind, MODE_STEP, a, launch, (cudaStream_t)stream);
}

int po_predict_dc(const po_hparams* hp, const float* w, const float* state1, const float* state2, float* w_hat,
                  int64_t n, const po_coef* coef_dev, const po_launch* launch, void* stream) {
  if (!valid_hp(hp) || coef_dev == nullptr) return PO_EINVAL;
  if (n > 0 && (w == nullptr || w_hat == nullptr || state1 == nullptr ||
                (hp->kind != PO_SGDM && state2 == nullptr)))
    return PO_EINVAL;
  Args a{const_cast<float*>(w), nullptr, const_cast<float*>(state1),
         hp->kind == PO_SGDM ? nullptr : const_cast<float*>(state2), w_hat, n, nullptr, coef_dev,
         coef(hp, 0.0, 0.0, 1)};
  return run(hp->kind, MODE_PREDICT, a, launch, (cudaStream_t)stream);
}

int po_step_predict_dc(const po_hparams* hp, float* w, const float* g, float* state1, float* state2,
                       float* w_hat, int64_t n, const po_coef* coef_dev, int64_t* nonfinite_index,
                       const po_launch* launch, void* stream) {
  if (!valid_hp(hp) || coef_dev == nullptr) return PO_EINVAL;
  if (n > 0 && (w == nullptr || g == nullptr || state1 == nullptr || w_hat == nullptr)) return PO_EINVAL;
  if (n > 0 && hp->kind != PO_SGDM && state2 == nullptr) return PO_EINVAL;
  Args a{w, g, state1, hp->kind == PO_SGDM ? nullptr : state2, w_hat, n,
         reinterpret_cast<unsigned long long*>(nonfinite_index), coef_dev, coef(hp, 0.0, 0.0, 1)};
  return run(hp->kind, MODE_STEP_PREDICT, a, launch, (cudaStream_t)stream);
}

int po_dp_signal(long long* const* peer_flag_slots, int32_t dp, int64_t epoch, void* stream) {
  if (peer_flag_slots == nullptr || dp < 1 || dp > kMaxDp) return PO_EINVAL;
  po_dp_signal_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(peer_flag_slots, dp, (long long)epoch, nullptr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

int po_dp_signal_dev(long long* const* peer_flag_slots, int32_t dp, int64_t* epoch_ctr, void* stream) {
  if (peer_flag_slots == nullptr || dp < 1 || dp > kMaxDp || epoch_ctr == nullptr) return PO_EINVAL;
  po_dp_signal_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(peer_flag_slots, dp, 0,
                                                          reinterpret_cast<long long*>(epoch_ctr));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

static int step_predict_dp_impl(const po_hparams* hp, float* w, const float* const* grads_host, int32_t dp,
                                float* state1, float* state2, float* w_hat, int64_t n, double lr,
                                double lr_pred_times_s, int64_t step_count, const po_coef* coef_dev,
                                int64_t* nonfinite_index, const int64_t* flags, int64_t epoch,
                                const int64_t* epoch_dev, int64_t timeout_ms, int32_t* status, void* stream);

int po_step_predict_dp(const po_hparams* hp, float* w, const float* const* grads_host, int32_t dp, float* state1,
                       float* state2, float* w_hat, int64_t n, double lr, double lr_pred_times_s,
                       int64_t step_count, int64_t* nonfinite_index, const int64_t* flags, int64_t epoch,
                       int64_t timeout_ms, int32_t* status, void* stream) {
  if (step_count < 0) return PO_EINVAL;
  return step_predict_dp_impl(hp, w, grads_host, dp, state1, state2, w_hat, n, lr, lr_pred_times_s, step_count,
                              nullptr, nonfinite_index, flags, epoch, nullptr, timeout_ms, status, stream);
}

int po_step_predict_dp_dc(const po_hparams* hp, float* w, const float* const* grads_host, int32_t dp, float* state1,
                          float* state2, float* w_hat, int64_t n, const po_coef* coef_dev, int64_t* nonfinite_index,
                          const int64_t* flags, const int64_t* epoch_ctr, int64_t timeout_ms, int32_t* status,
                          void* stream) {
  if (coef_dev == nullptr || epoch_ctr == nullptr) return PO_EINVAL;
  return step_predict_dp_impl(hp, w, grads_host, dp, state1, state2, w_hat, n, 0.0, 0.0, 0, coef_dev,
                              nonfinite_index, flags, 0, epoch_ctr, timeout_ms, status, stream);
}

static int step_predict_dp_impl(const po_hparams* hp, float* w, const float* const* grads_host, int32_t dp,
                                float* state1, float* state2, float* w_hat, int64_t n, double lr,
                                double lr_pred_times_s, int64_t step_count, const po_coef* coef_dev,
                                int64_t* nonfinite_index, const int64_t* flags, int64_t epoch,
                                const int64_t* epoch_dev, int64_t timeout_ms, int32_t* status, void* stream) {
  if (!valid_hp(hp) || step_count < 0 || dp < 1 || dp > kMaxDp || grads_host == nullptr || flags == nullptr ||
      status == nullptr || n < 0)
    return PO_EINVAL;
  if (n > 0 && (w == nullptr || state1 == nullptr || w_hat == nullptr || (hp->kind != PO_SGDM && state2 == nullptr)))
    return PO_EINVAL;
  DpArgs d;
  memset(&d, 0, sizeof(d));
  d.a = Args{w, nullptr, state1, hp->kind == PO_SGDM ? nullptr : state2, w_hat, n,
             reinterpret_cast<unsigned long long*>(nonfinite_index), coef_dev,
             coef(hp, lr, lr_pred_times_s, step_count + 1)};
  for (int r = 0; r < dp; ++r) {
    if (n > 0 && grads_host[r] == nullptr) return PO_EINVAL;
    d.grads[r] = grads_host[r];
  }
  d.dp = dp;
  d.inv_dp = (float)(1.0 / (double)dp);
  d.flags = reinterpret_cast<const long long*>(flags);
  d.epoch = (long long)epoch;
  d.timeout_cycles = (long long)(timeout_ms > 0 ? timeout_ms : 60000) * 2000000LL;  // ~2 GHz SM clock
  d.status = status;
  if (n == 0) return 0;
  int vec = 8;
  const void* ptrs[4] = {w, state1, hp->kind == PO_SGDM ? nullptr : state2, w_hat};
  auto all_aligned = [&](int bytes) {
    for (const void* p : ptrs)
      if (!aligned(p, bytes)) return false;
    for (int r = 0; r < dp; ++r)
      if (!aligned(grads_host[r], bytes)) return false;
    return true;
  };
  while (vec > 1 && !all_aligned(vec * 4)) vec = vec == 8 ? 4 : 1;
  // K3's launch shape for this size (block x CTAs/SM); one vector per stream
  // in flight, dp of them for the gradient
  // (large sizes: K3's 320 x 1 CTA/SM with the prefetching loop for dp <= 2,
  // 512 x 1 with one vector in flight above — the dp gradient loads are then
  // the requests in flight)
  const DefaultShape ds = n < (int64_t(1) << 25) ? default_shape(hp->kind, MODE_STEP_PREDICT, n)
                          : dp <= 2             ? DefaultShape{320, 1, 3, 1}
                                                : DefaultShape{512, 1, 1, 1};
  const int block = ds.block;
  const int64_t nv = n / vec;
  int64_t want = (nv + block - 1) / block;
  if (want < 1) want = 1;
  int64_t cap = (int64_t)sm_count() * ds.ctas_per_sm;
  const int64_t grid = want < cap ? want : cap;
  po_dp_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d.flags, dp, d.epoch, d.timeout_cycles, status,
                                                        reinterpret_cast<const long long*>(epoch_dev));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  switch (hp->kind) {
    case PO_SGDM: e = launch_dp<PO_SGDM>(d, vec, dim3((unsigned)grid), dim3(block), (cudaStream_t)stream); break;
    case PO_ADAM: e = launch_dp<PO_ADAM>(d, vec, dim3((unsigned)grid), dim3(block), (cudaStream_t)stream); break;
    default: e = launch_dp<PO_ADAMW>(d, vec, dim3((unsigned)grid), dim3(block), (cudaStream_t)stream); break;
  }
  return e == cudaSuccess ? 0 : (int)e;
}


int po_dp_shard_range(int64_t n, int32_t dp, int32_t rank, int64_t* lo, int64_t* hi) {
  if (n < 0 || dp < 1 || dp > kMaxDp || rank < 0 || rank >= dp || lo == nullptr || hi == nullptr) return PO_EINVAL;
  // contiguous shards of ceil(n / dp) rounded up to 64 elements (256 B), so
  // every shard but the last starts and ends on a 256-bit vector boundary
  int64_t chunk = (n + dp - 1) / dp;
  chunk = (chunk + 63) / 64 * 64;
  int64_t a = (int64_t)rank * chunk, b = a + chunk;
  if (a > n) a = n;
  if (b > n) b = n;
  *lo = a;
  *hi = b;
  return 0;
}

int po_step_predict_dp_shard(const po_hparams* hp, int32_t dp, int32_t rank, float* const* w, const float* const* grads,
                             float* const* state1, float* const* state2, float* const* w_hat, int64_t n, double lr,
                             double lr_pred_times_s, int64_t step_count, const po_coef* coef_dev,
                             int64_t* const* nonfinite_index, const int64_t* grad_flags, int64_t* const* done_slots,
                             const int64_t* done_flags, int64_t epoch, const int64_t* epoch_dev, int64_t timeout_ms,
                             int32_t* status, const po_dp_multicast* mc, void* stream) {
  if (!valid_hp(hp) || step_count < 0 || dp < 1 || dp > kMaxDp || rank < 0 || rank >= dp || n < 0 ||
      w == nullptr || grads == nullptr || state1 == nullptr || grad_flags == nullptr || done_slots == nullptr ||
      done_flags == nullptr || status == nullptr)
    return PO_EINVAL;
  const bool sg = hp->kind == PO_SGDM;
  if (!sg && state2 == nullptr) return PO_EINVAL;
  const bool use_mc = mc != nullptr && mc->grad != nullptr;
  if (use_mc && (mc->w == nullptr || mc->state1 == nullptr || (!sg && mc->state2 == nullptr) ||
                 ((w_hat != nullptr) != (mc->w_hat != nullptr))))
    return PO_EINVAL;
  DpShardArgs d;
  memset(&d, 0, sizeof(d));
  d.a = Args{nullptr, nullptr, nullptr, nullptr, nullptr, n, nullptr, coef_dev,
             coef(hp, lr, lr_pred_times_s, step_count + 1)};
  for (int r = 0; r < dp; ++r) {
    if (n > 0 && (w[r] == nullptr || grads[r] == nullptr || state1[r] == nullptr || (!sg && state2[r] == nullptr) ||
                  (w_hat != nullptr && w_hat[r] == nullptr)))
      return PO_EINVAL;
    d.w[r] = w[r];
    d.grads[r] = grads[r];
    d.s1[r] = state1[r];
    d.s2[r] = sg ? nullptr : state2[r];
    d.out[r] = w_hat != nullptr ? w_hat[r] : nullptr;
    d.bad[r] = nonfinite_index != nullptr ? reinterpret_cast<unsigned long long*>(nonfinite_index[r]) : nullptr;
  }
  if (use_mc) {
    d.mc_g = mc->grad;
    d.mc_w = mc->w;
    d.mc_s1 = mc->state1;
    d.mc_s2 = sg ? nullptr : mc->state2;
    d.mc_out = mc->w_hat;
  }
  d.dp = dp;
  d.rank = rank;
  d.inv_dp = (float)(1.0 / (double)dp);
  d.status = status;
  po_dp_shard_range(n, dp, rank, &d.lo, &d.hi);
  const long long timeout_cycles = (long long)(timeout_ms > 0 ? timeout_ms : 60000) * 2000000LL;
  cudaStream_t s = (cudaStream_t)stream;
  // 1) every replica's gradient of this epoch is complete
  po_dp_wait_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const long long*>(grad_flags), dp, (long long)epoch,
                                     timeout_cycles, status, reinterpret_cast<const long long*>(epoch_dev));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  // 2) this replica's shard: reduce, K3, write to all replicas
  const int64_t len = d.hi - d.lo;
  if (len > 0) {
    int vec = 8;
    auto all_aligned = [&](int bytes) {
      for (int r = 0; r < dp; ++r)
        if (!aligned(d.w[r] + d.lo, bytes) || !aligned(d.grads[r] + d.lo, bytes) || !aligned(d.s1[r] + d.lo, bytes) ||
            !aligned(d.s2[r] ? d.s2[r] + d.lo : nullptr, bytes) || !aligned(d.out[r] ? d.out[r] + d.lo : nullptr, bytes))
          return false;
      const float* m[5] = {d.mc_g, d.mc_w, d.mc_s1, d.mc_s2, d.mc_out};
      for (const float* p : m)
        if (p != nullptr && !aligned(p + d.lo, bytes)) return false;
      return true;
    };
    while (vec > 1 && !all_aligned(vec * 4)) vec = vec == 8 ? 4 : 1;
    // K3's one-vector-in-flight shapes: many small CTAs below 2^25 elements
    // (pipeline stages), 512 x 1 CTA/SM above
    const bool small = len < (int64_t(1) << 25);
    const int block = small ? 128 : 512;
    int64_t want = (len / vec + block - 1) / block;
    if (want < 1) want = 1;
    const int64_t cap = (int64_t)sm_count() * (small ? 16 : 1);
    const int64_t grid = want < cap ? want : cap;
    switch (hp->kind) {
      case PO_SGDM: e = launch_shard<PO_SGDM>(d, vec, use_mc, dim3((unsigned)grid), dim3(block), s); break;
      case PO_ADAM: e = launch_shard<PO_ADAM>(d, vec, use_mc, dim3((unsigned)grid), dim3(block), s); break;
      default: e = launch_shard<PO_ADAMW>(d, vec, use_mc, dim3((unsigned)grid), dim3(block), s); break;
    }
    if (e != cudaSuccess) return (int)e;
  }
  // 3) announce this shard; 4) wait until every owner has written its shard here
  po_dp_done_kernel<<<1, 32, 0, s>>>(reinterpret_cast<long long* const*>(done_slots), dp, (long long)epoch,
                                     reinterpret_cast<const long long*>(epoch_dev), status);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  po_dp_wait_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const long long*>(done_flags), dp, (long long)epoch,
                                     timeout_cycles, status, reinterpret_cast<const long long*>(epoch_dev));
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
