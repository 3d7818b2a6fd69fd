// tma_stream_probe.cu — can TMA bulk copies (cp.async.bulk, global <-> shared,
// mbarrier-tracked loads, bulk-group stores) stream HBM faster than per-thread
// 256-bit LDG/STG? Times, at ~1e9 fp32 elements per stream:
//   copy_ldst   : persistent grid-stride 256-bit ld/st copy (the K3 loop shape)
//   copy_tma    : 1 in / 1 out stream through a shared-memory ring
//   k3_tma      : the fused Adam step + prediction (4 in / 4 out streams,
//                 computed in place in shared memory between the bulk load
//                 and the bulk store)
// for several tile sizes / ring depths; prints one JSON line per config.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream_probe scripts/tma_stream_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("FAIL %s: %s\n", #x, cudaGetErrorString(e_));                         \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n }" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct P {
  float* in[4];   // copy: in[0]; k3: w, g, m, v
  float* out[4];  // copy: out[0]; k3: w, m, v, w_hat
  long long n;    // elements per stream (multiple of TE)
  float lr, c_pred, ibc1, ibc2, b1, omb1, b2, omb2, eps;
};

__device__ __forceinline__ void adam_elem(const P& p, float& w, float g, float& m, float& v, float& wh) {
  m = __fadd_rn(__fmul_rn(p.b1, m), __fmul_rn(p.omb1, g));
  v = __fadd_rn(__fmul_rn(p.b2, v), __fmul_rn(p.omb2, __fmul_rn(g, g)));
  float d = __fdiv_rn(__fmul_rn(m, p.ibc1), __fadd_rn(__fsqrt_rn(__fmul_rn(v, p.ibc2)), p.eps));
  float nw = __fsub_rn(w, __fmul_rn(p.lr, d));
  w = nw;
  wh = __fsub_rn(nw, __fmul_rn(p.c_pred, d));
}

// OP 0: copy (1 stream in, 1 out). OP 1: K3 Adam (4 in, 4 out, in place).
template <int OP, int TE, int STAGES>
__global__ void __launch_bounds__(256, 1) tma_kernel(const P p) {
  constexpr int NS = OP == 0 ? 1 : 4;
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const int tid = threadIdx.x;
  const long long ntiles = p.n / TE;
  const long long my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto buf = [&](int st, int s) { return sm + ((size_t)st * NS + s) * TE; };
  auto issue_load = [&](long long k) {
    const int st = (int)(k % STAGES);
    const long long t = blockIdx.x + k * gridDim.x;
    mbar_expect_tx(&full[st], NS * TE * 4);
#pragma unroll
    for (int s = 0; s < NS; ++s) bulk_load(buf(st, s), p.in[s] + t * TE, TE * 4, &full[st]);
  };
  if (tid == 0)
    for (long long k = 0; k < STAGES && k < my; ++k) issue_load(k);
  for (long long k = 0; k < my; ++k) {
    const int st = (int)(k % STAGES);
    mbar_wait(&full[st], (uint32_t)((k / STAGES) & 1));
    if constexpr (OP == 1) {
      float4* W = (float4*)buf(st, 0);
      float4* G = (float4*)buf(st, 1);
      float4* M = (float4*)buf(st, 2);
      float4* V = (float4*)buf(st, 3);
#pragma unroll 2
      for (int e = tid; e < TE / 4; e += 256) {
        float4 w = W[e], g = G[e], m = M[e], v = V[e], wh;
        adam_elem(p, w.x, g.x, m.x, v.x, wh.x);
        adam_elem(p, w.y, g.y, m.y, v.y, wh.y);
        adam_elem(p, w.z, g.z, m.z, v.z, wh.z);
        adam_elem(p, w.w, g.w, m.w, v.w, wh.w);
        W[e] = w;
        M[e] = m;
        V[e] = v;
        G[e] = wh;  // W_hat takes the gradient's slot
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
      const long long t = blockIdx.x + k * gridDim.x;
      if constexpr (OP == 0) {
        bulk_store(p.out[0] + t * TE, buf(st, 0), TE * 4);
      } else {
        bulk_store(p.out[0] + t * TE, buf(st, 0), TE * 4);
        bulk_store(p.out[1] + t * TE, buf(st, 2), TE * 4);
        bulk_store(p.out[2] + t * TE, buf(st, 3), TE * 4);
        bulk_store(p.out[3] + t * TE, buf(st, 1), TE * 4);
      }
      bulk_commit();
      // refill the stage of tile k-1 once its stores have read shared memory
      if (k >= 1 && k - 1 + STAGES < my) {
        bulk_wait_read<1>();
        issue_load(k - 1 + STAGES);
      }
    }
  }
  if (tid == 0) bulk_wait_all();
}

__global__ void __launch_bounds__(512) copy_ldst(const float* __restrict__ a, float* __restrict__ b, long long n8) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
    float r0, r1, r2, r3, r4, r5, r6, r7;
    asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r0), "=f"(r1), "=f"(r2), "=f"(r3), "=f"(r4), "=f"(r5), "=f"(r6), "=f"(r7)
                 : "l"(a + 8 * i));
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(b + 8 * i), "f"(r0), "f"(r1),
                 "f"(r2), "f"(r3), "f"(r4), "f"(r5), "f"(r6), "f"(r7)
                 : "memory");
  }
}

template <typename F>
float time_ms(F f, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 2; ++i) f();
  float best = 1e30f, tot = 0;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
    tot += ms;
  }
  return tot / reps;
}

template <int OP, int TE, int STAGES>
int run_tma(P p, int sms, long long n_elems, int reps) {
  constexpr int NS = OP == 0 ? 1 : 4;
  const int smem = STAGES * NS * TE * 4;
  auto k = tma_kernel<OP, TE, STAGES>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  p.n = n_elems / TE * TE;
  float ms = time_ms([&] { k<<<sms, 256, smem>>>(p); }, reps);
  CK(cudaGetLastError());
  double bytes = (double)p.n * 4 * NS * 2;
  printf("{\"kernel\": \"%s\", \"te\": %d, \"stages\": %d, \"smem\": %d, \"n\": %lld, \"ms\": %.4f, \"gbs\": %.1f}\n",
         OP == 0 ? "copy_tma" : "k3_adam_tma", TE, STAGES, smem, p.n, ms, bytes / ms / 1e6);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long n = 1000000000LL;
  float* buf[6];
  for (int i = 0; i < 6; ++i) {
    CK(cudaMalloc(&buf[i], n * 4));
    CK(cudaMemset(buf[i], 0, n * 4));
  }
  const int reps = 10;
  {
    float ms = time_ms([&] { cudaMemcpyAsync(buf[1], buf[0], n * 4, cudaMemcpyDeviceToDevice); }, reps);
    printf("{\"kernel\": \"cudaMemcpy_d2d\", \"n\": %lld, \"ms\": %.4f, \"gbs\": %.1f}\n", n, ms, 8.0 * n / ms / 1e6);
    for (int cps : {1, 2, 4}) {
      for (int blk : {256, 512}) {
        float ms2 = time_ms([&] { copy_ldst<<<sms * cps, blk>>>(buf[0], buf[1], n / 8); }, reps);
        printf("{\"kernel\": \"copy_ldst\", \"ctas_per_sm\": %d, \"block\": %d, \"n\": %lld, \"ms\": %.4f, \"gbs\": %.1f}\n",
               cps, blk, n, ms2, 8.0 * n / ms2 / 1e6);
      }
    }
  }
  P p{};
  p.in[0] = buf[0];
  p.out[0] = buf[1];
  run_tma<0, 4096, 4>(p, sms, n, reps);
  run_tma<0, 8192, 4>(p, sms, n, reps);
  run_tma<0, 8192, 6>(p, sms, n, reps);
  run_tma<0, 16384, 3>(p, sms, n, reps);
  // K3: w g m v in; w m v w_hat out (in place + w_hat)
  P q{};
  q.in[0] = buf[0];
  q.in[1] = buf[1];
  q.in[2] = buf[2];
  q.in[3] = buf[3];
  q.out[0] = buf[0];
  q.out[1] = buf[2];
  q.out[2] = buf[3];
  q.out[3] = buf[4];
  q.lr = 1e-3f;
  q.c_pred = 3e-3f;
  q.ibc1 = 10.f;
  q.ibc2 = 100.f;
  q.b1 = 0.9f;
  q.omb1 = 0.1f;
  q.b2 = 0.999f;
  q.omb2 = 0.001f;
  q.eps = 1e-8f;
  run_tma<1, 1024, 4>(q, sms, n, reps);
  run_tma<1, 1024, 6>(q, sms, n, reps);
  run_tma<1, 2048, 3>(q, sms, n, reps);
  run_tma<1, 2048, 4>(q, sms, n, reps);
  run_tma<1, 2048, 6>(q, sms, n, reps);
  run_tma<1, 4096, 3>(q, sms, n, reps);
  CK(cudaDeviceSynchronize());
  return 0;
}
