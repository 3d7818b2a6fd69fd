// pipeoptim_wgrad.cu — the weight gradient of an MLP layer computed on the
// tcgen05 tensor cores with the optimizer update (K2, or K3 = step + next
// forward's prediction) applied in the GEMM's epilogue.
//
// In 1F1B every backward B_j of a stage is immediately followed by its update
// U_j (stages.py:187-209 then runtime.py:449-463). Unfused, the weight
// gradient GEMM writes dW (4 B/param) and K3 reads it back; here the fp32
// accumulator tile goes from TMEM straight into the update: per parameter the
// kernel moves W, m, v in and W', m', v', W_hat out (28 B Adam, K3) instead of
// 4 + 32, and the stage's B→U chain loses a launch.
//
//   dW (in x out) = x^T (in x rows) @ dpre (rows x out)
//
// x (rows x in) and dpre (rows x out) are row-major activations; `rows` (the
// micro-batch) is the GEMM's K. One CTA per 128 x 64 output tile, 8 warps:
//   1. the warps load a 64-deep K chunk of both operands (16-byte loads along
//      in / out, all of a thread's loads in flight together), split each value
//      into three bf16 pieces
//      (a = a0 + a1 + a2 exactly to 24 bits) and store the pieces in shared
//      memory (3xTF32 by default: two fp32 pieces, see kTf32) in the UMMA
//      canonical K-major, no-swizzle layout (8-row x 16-byte
//      core matrices; LBO 128 B between the two K halves of an MMA, SBO
//      1 KB + 16 B between 8-row groups, which spreads a warp's stores over
//      all bank groups);
//   2. one thread issues tcgen05.mma.kind::f16 (M = 128, N = 64, K = 16) for the
//      six piece products that carry 24-bit accuracy (a2b0 + a1b1 + a0b2 +
//      a1b0 + a0b1 + a0b0, smallest first), accumulating in fp32 in TMEM, and
//      commits to an mbarrier;
//   3. after the last chunk each warp copies its TMEM lane quadrant (32 rows)
//      and column half (tcgen05.ld.32x32b) into shared memory, then the warps
//      walk the tile two rows per step (W / m / v of the first step loaded
//      before waiting for the MMAs, each step prefetching the next) applying
//      the shared per-element rule (pipeoptim_rules.cuh) — every W / m / v /
//      W_hat access of a half-warp one contiguous 256-byte segment.
//
// Measured (scripts/wgrad_kernel_bench.py, graph-timed, L2 warm; the
// variants in profiles/r2_wgrad_fused_bench.jsonl): with the 3xTF32 split,
// config-1 stage 0 (128 x 3072 x 1024) 23.5 us vs 26.2 us for the split-K
// tensor-core GEMM + K3, stages 1-2 (128 x 1024 x 1024) 10.4 vs 12.4 us
// (bf16x3: 27.1 / 12.3 — its in-tile split cost ~6 us). In config 1's
// single-GPU 1F1B run (profiles/r2_wgrad_fusion_pipeline_ab_3xtf32.jsonl) it
// lifts prediction-off throughput 6 % but prediction-on only 2 %, the
// prediction overhead rises from 1.9 % to 5.2 % and the per-stage unit times
// do not improve, so stages.FUSE_WGRAD_UPDATE stays off by default (and the
// path is for fp32 runs: with TF32 GEMMs allowed the library TF32 GEMM is
// cheaper than 3xTF32). With programmatic dependent launch (prologue over
// the previous kernel's tail) the 1F1B run gains 4.4 % with prediction on
// (7.4 % off) at a 4.95 % overhead, but the stage-0 unit (the one-stage-per-
// GPU bound) is still 48 / 51.5 us vs 45 / 47 us unfused: the 384 tiles
// take 1.3 waves of 2 CTAs / SM, a latency the persistent GEMM + K3 avoid.
// A 4-warp, 4-CTAs/SM variant (one wave) was slower (26.4 / 12.9 us).
// A warp-specialised persistent form (one CTA per SM:
// 4 producer warps, one MMA thread, 4 epilogue warps on two TMEM
// accumulators, so a tile's update overlaps the next tile's loads and MMAs)
// was slower — 44.5 / 18.8 us: one CTA's 4 + 4 warps have a quarter of the
// split throughput and memory parallelism of two 8-warp CTAs — and was
// dropped.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "pipeoptim.h"
#include "pipeoptim_rules.cuh"

namespace {

constexpr int kTM = 128;                       // output tile rows (in); the MMA's M
constexpr int kTN = 64;                        // output tile columns (out); the MMA's N
constexpr int kKC = 64;                        // K chunk staged in shared memory
constexpr int kThreads = 256;                  // 8 warps: 2 per TMEM lane quadrant
// 8-row group stride: the (kKC / 8) 128-byte core matrices of a group plus 16
// bytes, so the 16-byte stores of a warp (rows 4 apart) hit all 8 bank groups
// Operand precision split (compile-time): 3xTF32 (default) — a = big + small
// with big = tf32(a) and small = a - big exactly, products big*big +
// big*small + small*big on tcgen05.mma.kind::tf32 — or bf16x3 (three bf16
// pieces, six products on kind::f16). 3xTF32 costs two instructions per
// element to split (bf16x3 ~10) and half the MMAs.
#ifndef PO_WGRAD_BF16X3
constexpr bool kTf32 = true;
#else
constexpr bool kTf32 = false;
#endif
constexpr int kPieces = kTf32 ? 2 : 3;
constexpr int kElemsPerChunk = kTf32 ? 4 : 8;  // operand elements per 16-byte core-matrix row
constexpr int kMmaK = kTf32 ? 8 : 16;          // K of one MMA (32 bytes of each operand row)
// 8-row group stride: the core matrices along K plus 16 bytes, so the
// 16-byte stores of a warp (rows 4 apart) hit all 8 bank groups
constexpr uint32_t kSBO = (kKC / kElemsPerChunk) * 128 + 16;
constexpr uint32_t kLBO = 128;                 // K-chunk stride within one MMA (bytes)
constexpr int kPieceA = (kTM / 8) * kSBO;      // one piece of the A chunk
constexpr int kPieceB = (kTN / 8) * kSBO;      // one piece of the B chunk
constexpr int kOperands = kPieces * (kPieceA + kPieceB);  // 99 KB (3xTF32) / 73 KB (bf16x3)
constexpr int kSmem = kOperands;               // 2 CTAs / SM
constexpr uint32_t kTmemCols = kTN;            // fp32 accumulator columns
constexpr int kTS = kTN + 4;                   // epilogue tile row stride (floats)
static_assert(kTM * kTS * 4 <= kOperands, "the epilogue's accumulator tile reuses the operand buffers");

struct WgradArgs {
  const float* x;
  int64_t ldx;
  const float* dpre;
  int64_t ldd;
  int64_t rows, in, out;
  float* w;
  float* s1;
  float* s2;
  float* w_hat;  // null: K2
  float* g_out;  // nullable: also store the gradient
  unsigned long long* bad;
  int64_t flat_offset;
  const po_coef* dc;
  Coef c;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (cute::UMMA::SmemDescriptor):
// start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((kLBO >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((kSBO >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// instruction descriptor (cute::UMMA::InstrDescriptor): D f32 [4,6), A and B
// format [7,10) / [10,13) (1 = BF16, 2 = TF32), both K-major, N >> 3
// [17,23), M >> 4 [24,29)
constexpr uint32_t kFmt = kTf32 ? 2u : 1u;
constexpr uint32_t kIdesc = (1u << 4) | (kFmt << 7) | (kFmt << 10) | ((uint32_t)(kTN >> 3) << 17) |
                            ((uint32_t)(kTM >> 4) << 24);

__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  if constexpr (kTf32)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n }" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// byte offset of (row r, K group g of 8) in one piece: canonical K-major core matrices
__device__ __forceinline__ uint32_t core_off(int r, int g) {
  return (uint32_t)(r >> 3) * kSBO + (uint32_t)g * 128u + (uint32_t)(r & 7) * 16u;
}

// 3xTF32 pieces of 4 consecutive K elements of one operand row: big =
// tf32(a) (round to nearest), small = a - big (exact in fp32; the MMA reads
// its top 19 bits)
__device__ __forceinline__ void split_store_tf32(const float (&v)[4], uint8_t* base, uint32_t off, int piece) {
  uint32_t big[4], small[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(big[j]) : "f"(v[j]));
    small[j] = __float_as_uint(__fsub_rn(v[j], __uint_as_float(big[j])));
  }
  *reinterpret_cast<uint4*>(base + off) = make_uint4(big[0], big[1], big[2], big[3]);
  *reinterpret_cast<uint4*>(base + piece + off) = make_uint4(small[0], small[1], small[2], small[3]);
}

[[maybe_unused]] __device__ __forceinline__ void split_store(const float (&v)[8], uint8_t* base, uint32_t off,
                                                            int piece) {
#ifdef PO_PROBE_NO_SPLIT  // timing probe only: the operand split's cost (results are wrong)
  *reinterpret_cast<uint4*>(base + off) = make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                                                     __float_as_uint(v[2]), __float_as_uint(v[3]));
  return;
#endif
  uint32_t p0[4], p1[4], p2[4];
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    __nv_bfloat16 h[2], m[2], l[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float a = v[j + u];
      h[u] = __float2bfloat16_rn(a);
      const float r1 = __fsub_rn(a, __bfloat162float(h[u]));
      m[u] = __float2bfloat16_rn(r1);
      l[u] = __float2bfloat16_rn(__fsub_rn(r1, __bfloat162float(m[u])));
    }
    p0[j / 2] = (uint32_t)__bfloat16_as_ushort(h[0]) | ((uint32_t)__bfloat16_as_ushort(h[1]) << 16);
    p1[j / 2] = (uint32_t)__bfloat16_as_ushort(m[0]) | ((uint32_t)__bfloat16_as_ushort(m[1]) << 16);
    p2[j / 2] = (uint32_t)__bfloat16_as_ushort(l[0]) | ((uint32_t)__bfloat16_as_ushort(l[1]) << 16);
  }
  *reinterpret_cast<uint4*>(base + off) = make_uint4(p0[0], p0[1], p0[2], p0[3]);
  *reinterpret_cast<uint4*>(base + piece + off) = make_uint4(p1[0], p1[1], p1[2], p1[3]);
  *reinterpret_cast<uint4*>(base + 2 * piece + off) = make_uint4(p2[0], p2[1], p2[2], p2[3]);
}

template <int KIND, bool PREDICT>
__global__ void __launch_bounds__(kThreads, 2) wgrad_update_kernel(const WgradArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                      // the pieces of x^T (rows = in)
  uint8_t* sB = smem + kPieces * kPieceA;  // the pieces of dpre^T (rows = out)
  __shared__ __align__(8) uint64_t mma_bar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.y * kTM, n0 = (int64_t)blockIdx.x * kTN;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mma_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  // programmatic dependent launch: the set-up above overlapped the previous
  // kernel's tail; everything it may have written is read only after this
  // (a no-op when the launch carried no PDL attribute)
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const int nchunks = (int)((a.rows + kKC - 1) / kKC);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int64_t k0 = (int64_t)ch * kKC;
    const int kc = (int)(a.rows - k0 < kKC ? a.rows - k0 : kKC);  // a multiple of 16
    if (ch > 0) mbar_wait(&mma_bar, (uint32_t)((ch - 1) & 1));     // the MMAs read the previous chunk
    // warp w loads K group w (8 rows of k): lane l the 4 consecutive A rows
    // 4l..4l+3 (16-byte loads, 512 B per warp and k row) and, on lanes 0-15,
    // the 4 B rows 4l..4l+3; all loads in flight before the first split
    if (warp < kc / 8) {
      const int64_t kb = k0 + 8 * warp;
      const bool bl = lane < kTN / 4;
      float4 av[8], bv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        av[j] = __ldg(reinterpret_cast<const float4*>(a.x + (kb + j) * a.ldx + m0) + lane);
        if (bl) bv[j] = __ldg(reinterpret_cast<const float4*>(a.dpre + (kb + j) * a.ldd + n0) + lane);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float ca[8], cb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          ca[j] = u == 0 ? av[j].x : u == 1 ? av[j].y : u == 2 ? av[j].z : av[j].w;
          cb[j] = u == 0 ? bv[j].x : u == 1 ? bv[j].y : u == 2 ? bv[j].z : bv[j].w;
        }
        if constexpr (kTf32) {  // two 4-element K chunks (2w, 2w + 1) per row
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float qa[4] = {ca[4 * h], ca[4 * h + 1], ca[4 * h + 2], ca[4 * h + 3]};
            const float qb[4] = {cb[4 * h], cb[4 * h + 1], cb[4 * h + 2], cb[4 * h + 3]};
            split_store_tf32(qa, sA, core_off(4 * lane + u, 2 * warp + h), kPieceA);
            if (bl) split_store_tf32(qb, sB, core_off(4 * lane + u, 2 * warp + h), kPieceB);
          }
        } else {
          split_store(ca, sA, core_off(4 * lane + u, warp), kPieceA);
          if (bl) split_store(cb, sB, core_off(4 * lane + u, warp), kPieceB);
        }
      }
    }
    // generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      // (A piece, B piece) products carrying fp32-level accuracy, smallest
      // first: 3xTF32 small*big, big*small, big*big; bf16x3 the six of
      // a2b0 + a1b1 + a0b2 + a1b0 + a0b1 + a0b0
      constexpr int kProducts = kTf32 ? 3 : 6;
      constexpr int pa[6] = {kTf32 ? 1 : 2, kTf32 ? 0 : 1, 0, 1, 0, 0};
      constexpr int pb[6] = {0, kTf32 ? 1 : 1, kTf32 ? 0 : 2, 0, 1, 0};
      for (int s = 0; s < kc / kMmaK; ++s) {
#pragma unroll
        for (int p = 0; p < kProducts; ++p) {
          const uint64_t da = smem_desc(a0 + (uint32_t)(pa[p] * kPieceA) + (uint32_t)s * 256u);
          const uint64_t db = smem_desc(b0 + (uint32_t)(pb[p] * kPieceB) + (uint32_t)s * 256u);
          mma(tmem, da, db, (ch > 0 || s > 0 || p > 0) ? 1u : 0u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&mma_bar))
                   : "memory");
    }
  }

  // ---- epilogue ----
  // The update walks the tile two rows per warp step (half-warp h takes row
  // 2t + h, lane l % 16 columns 4(l % 16)..+3): every W / m / v / W_hat access
  // of a half-warp is one contiguous 256-byte segment. W / m / v do not depend
  // on the GEMM: the first step's loads are issued before waiting for the
  // MMAs, and each step prefetches the next.
  Coef c = a.c;
  if (a.dc != nullptr) {
    const po_coef d = *a.dc;
    c.lr = d.lr;
    c.c_pred = d.c_pred;
    c.ibc1 = d.inv_bc1;
    c.ibc2 = d.inv_bc2;
  }
  constexpr int kRowsPerWarp = kTM / (kThreads / 32);  // 16
  const int hw = lane >> 4, col = 4 * (lane & 15);
  auto fidx = [&](int t) { return (m0 + warp * kRowsPerWarp + 2 * t + hw) * a.out + n0 + col; };
  float4 w = __ldcs(reinterpret_cast<const float4*>(a.w + fidx(0)));
  float4 s1 = __ldcs(reinterpret_cast<const float4*>(a.s1 + fidx(0)));
  float4 s2 = make_float4(0.f, 0.f, 0.f, 0.f);
  if constexpr (KIND != PO_SGDM) s2 = __ldcs(reinterpret_cast<const float4*>(a.s2 + fidx(0)));

  mbar_wait(&mma_bar, (uint32_t)((nchunks - 1) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // the next kernel may be scheduled now (its own griddepcontrol.wait still
  // waits for this grid to complete)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // TMEM -> shared memory: warp w reads lane quadrant w % 4 (32 rows) and
  // column half w / 4; the operand buffers are free once the MMAs completed
  float* tile = reinterpret_cast<float*>(smem);
  {
    const int quad = warp & 3, half = warp >> 2;
    const int trow = quad * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * (kTN / 2));
#pragma unroll
    for (int q = 0; q < kTN / 2; q += 16) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr + (uint32_t)q));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float4* dst = reinterpret_cast<float4*>(tile + trow * kTS + half * (kTN / 2) + q);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        dst[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]), __uint_as_float(r[4 * v + 2]),
                             __uint_as_float(r[4 * v + 3]));
    }
  }
  __syncthreads();
  int64_t bad = INT64_MAX;
  for (int t = 0; t < kRowsPerWarp / 2; ++t) {
    const int64_t f = fidx(t);
    float4 nw{}, ns1{}, ns2{};
    if (t + 1 < kRowsPerWarp / 2) {  // prefetch the next step
      const int64_t fn = fidx(t + 1);
      nw = __ldcs(reinterpret_cast<const float4*>(a.w + fn));
      ns1 = __ldcs(reinterpret_cast<const float4*>(a.s1 + fn));
      if constexpr (KIND != PO_SGDM) ns2 = __ldcs(reinterpret_cast<const float4*>(a.s2 + fn));
    }
    float4 g = *reinterpret_cast<const float4*>(tile + (warp * kRowsPerWarp + 2 * t + hw) * kTS + col);
    float4 o;
    float* wp = &w.x;
    float* m1 = &s1.x;
    float* m2 = &s2.x;
    float* gp = &g.x;
    float* op = &o.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      bool e = false;
      elem<KIND, PREDICT ? MODE_STEP_PREDICT : MODE_STEP>(c, wp[j], gp[j], m1[j], KIND != PO_SGDM ? m2[j] : m1[j],
                                                          op[j], e);
      if (e && bad == INT64_MAX) bad = a.flat_offset + f + j;
    }
    __stcs(reinterpret_cast<float4*>(a.w + f), w);
    __stcs(reinterpret_cast<float4*>(a.s1 + f), s1);
    if constexpr (KIND != PO_SGDM) __stcs(reinterpret_cast<float4*>(a.s2 + f), s2);
    if constexpr (PREDICT) __stcs(reinterpret_cast<float4*>(a.w_hat + f), o);
    if (a.g_out != nullptr) __stcs(reinterpret_cast<float4*>(a.g_out + f), g);
    w = nw;
    s1 = ns1;
    s2 = ns2;
  }
  if (a.bad != nullptr && bad != INT64_MAX) atomicMin(a.bad, (unsigned long long)bad);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

// launched with programmatic dependent launch (its prologue — TMEM alloc,
// barrier init — overlaps the previous kernel), like the library GEMMs
#ifndef PO_WGRAD_NO_PDL
constexpr bool kWgradPdl = true;
#else
constexpr bool kWgradPdl = false;
#endif

template <int KIND, bool PREDICT>
cudaError_t launch(const WgradArgs& a, cudaStream_t s) {
  // the dynamic shared-memory opt-in (> 48 KB), once per instantiation
  // (thread-safe static initialisation)
  static const cudaError_t attr = cudaFuncSetAttribute(wgrad_update_kernel<KIND, PREDICT>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  if (attr != cudaSuccess) return attr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.out / kTN), (unsigned)(a.in / kTM));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = kWgradPdl ? 1 : 0;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, wgrad_update_kernel<KIND, PREDICT>, a);
}

bool aligned32(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 31) == 0; }

}  // namespace

extern "C" {

int po_wgrad_update_supported(int64_t rows, int64_t in, int64_t out) {
  return rows >= 16 && rows % 16 == 0 && in >= kTM && in % kTM == 0 && out >= kTN && out % kTN == 0 &&
         in / kTM <= 65535;
}

int po_wgrad_update(const po_hparams* hp, const float* x, int64_t ldx, const float* dpre, int64_t ldd, int64_t rows,
                    int64_t in, int64_t out, float* w, float* state1, float* state2, float* w_hat, float* g_out,
                    double lr, double lr_pred_times_s, int64_t step_count, const po_coef* coef_dev,
                    int64_t* nonfinite_index, int64_t flat_offset, void* stream) {
  if (hp == nullptr || (hp->kind != PO_SGDM && hp->kind != PO_ADAM && hp->kind != PO_ADAMW) || step_count < 0)
    return PO_EINVAL;
  if (!po_wgrad_update_supported(rows, in, out) || x == nullptr || dpre == nullptr || w == nullptr ||
      state1 == nullptr || (hp->kind != PO_SGDM && state2 == nullptr) || ldx < in || ldd < out || ldx % 4 ||
      ldd % 4 || flat_offset < 0)
    return PO_EINVAL;
  const void* vec[5] = {w, state1, state2, w_hat, g_out};
  for (const void* p : vec)
    if (!aligned32(p)) return PO_EINVAL;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(dpre) & 15)) return PO_EINVAL;
  WgradArgs a;
  memset(&a, 0, sizeof(a));
  a.x = x;
  a.ldx = ldx;
  a.dpre = dpre;
  a.ldd = ldd;
  a.rows = rows;
  a.in = in;
  a.out = out;
  a.w = w;
  a.s1 = state1;
  a.s2 = hp->kind == PO_SGDM ? nullptr : state2;
  a.w_hat = w_hat;
  a.g_out = g_out;
  a.bad = reinterpret_cast<unsigned long long*>(nonfinite_index);
  a.flat_offset = flat_offset;
  a.dc = coef_dev;
  // K3: the step at t = step_count + 1 and the read right after it (S5);
  // K2: the step alone (same coefficients)
  a.c = coef(hp, lr, lr_pred_times_s, step_count + 1);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  const bool pred = w_hat != nullptr;
  switch (hp->kind) {
    case PO_SGDM: e = pred ? launch<PO_SGDM, true>(a, s) : launch<PO_SGDM, false>(a, s); break;
    case PO_ADAM: e = pred ? launch<PO_ADAM, true>(a, s) : launch<PO_ADAM, false>(a, s); break;
    default: e = pred ? launch<PO_ADAMW, true>(a, s) : launch<PO_ADAMW, false>(a, s); break;
  }
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
