// pipeoptim_p2p.cu — peer-memory transport for the 1F1B boundary tensors.
//
// The pipeline's only exchange is neighbour point-to-point: the activation of
// mini-batch m moves stage k -> k+1 after F(m, k), its input gradient
// k+1 -> k after B(m, k+1). Instead of NCCL send/recv driven
// by the host, each direction is a ring of `slots` message buffers that lives
// on the RECEIVING GPU and is mapped into the sender (CUDA IPC; NVLink /
// NVSwitch peer memory on a multi-GPU node):
//
//   sender:   wait until the receiver has acknowledged message sent+1-slots
//             (ring credit), store the tensor straight into ring[sent % slots]
//             on the peer, then release-store ready = sent+1 on the peer.
//   receiver: wait until ready >= recvd+1, copy ring[recvd % slots] into the
//             op's static input buffer, then release-store ack = recvd+1 on
//             the sender.
//
// Every counter lives in device memory and is advanced by the kernels
// themselves, so the host never takes part: a rank's whole 1F1B program
// (sends, receives, stage math, optimizer) is ONE stream of work that can be
// captured into ONE CUDA graph and replayed, the flags carrying the
// cross-GPU ordering. Waits are a single 32-thread CTA (never a full-grid
// spin that could starve the GPU's other work), bounded by a timeout that
// sets *status and lets the run finish instead of hanging; the host raises.
//
// Control block (int64 x 4, local to each rank, zero-initialised):
//   ctl[0] messages sent      ctl[1] arrival counter of the send copy kernel
//   ctl[2] messages received  ctl[3] arrival counter of the receive copy kernel
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "pipeoptim.h"

namespace {

__device__ __forceinline__ long long p2p_ld_acquire(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void p2p_st_release(long long* p, long long v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Wait until *flag >= *ctr + 1 - lag (lag = slots for the send credit, 0 for
// a receive). One thread polls; on timeout *status = 1.
__global__ void p2p_wait_kernel(const long long* flag, const long long* ctr, long long lag, long long timeout_cycles,
                                int* status) {
  if (threadIdx.x != 0) return;
  if (*(volatile int*)status != 0) return;
  const long long target = *(volatile const long long*)ctr + 1 - lag;
  const long long t0 = clock64();
  while (p2p_ld_acquire(flag) < target) {
    if (clock64() - t0 > timeout_cycles) {
      atomicExch(status, 1);
      return;
    }
    __nanosleep(256);
  }
}

// Copy n floats src -> dst where ONE side is ring[ctr % slots]; then the last
// CTA to finish advances *ctr and release-stores the new count into *flag
// (the peer's ready flag for a send, the peer's ack flag for a receive).
template <bool RING_IS_DST>
__global__ void p2p_copy_signal_kernel(const float* src, float* dst, int64_t n, int64_t slot_elems, int slots,
                                       long long* ctr, unsigned long long* arrive, long long* flag, const int* status) {
  __shared__ bool last;
  const bool failed = *(volatile const int*)status != 0;
  const long long c = *(volatile long long*)ctr;
  const int64_t off = (int64_t)(c % slots) * slot_elems;
  const float* s = RING_IS_DST ? src : src + off;
  float* d = RING_IS_DST ? dst + off : dst;
  if (!failed) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0;
    const int64_t n4 = vec ? n / 4 : 0;
    const float4* s4 = reinterpret_cast<const float4*>(s);
    float4* d4 = reinterpret_cast<float4*>(d);
    for (int64_t i = tid; i < n4; i += stride) d4[i] = s4[i];
    for (int64_t i = n4 * 4 + tid; i < n; i += stride) d[i] = s[i];
  }
  __threadfence_system();  // this CTA's stores (peer memory for a send) before its arrival
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(arrive, 1ull) == (unsigned long long)(gridDim.x - 1);
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    *arrive = 0ull;  // re-armed for the next message (graph replays)
    if (!failed) {
      *ctr = c + 1;
      p2p_st_release(flag, c + 1);
    }
  }
}

int p2p_grid(int64_t n) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms = v > 0 ? v : 148;
  }
  const int64_t want = (n / 4 + 255) / 256;
  const int64_t cap = (int64_t)sms * 2;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

long long cycles(int64_t timeout_ms) { return (long long)(timeout_ms > 0 ? timeout_ms : 60000) * 2000000LL; }

}  // namespace

extern "C" {

int po_p2p_send(const float* src, int64_t n, float* peer_ring, int64_t slot_elems, int32_t slots, int64_t* ctl,
                const int64_t* ack_flag, int64_t* peer_ready_flag, int64_t timeout_ms, int32_t* status,
                void* stream) {
  if (n < 0 || slots < 1 || slot_elems < n || ctl == nullptr || ack_flag == nullptr || peer_ready_flag == nullptr ||
      status == nullptr || peer_ring == nullptr || (n > 0 && src == nullptr) || (slot_elems & 3) != 0)
    return PO_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  long long* c = reinterpret_cast<long long*>(ctl);
  p2p_wait_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const long long*>(ack_flag), c, slots, cycles(timeout_ms),
                                   status);
  p2p_copy_signal_kernel<true><<<p2p_grid(n), 256, 0, s>>>(src, peer_ring, n, slot_elems, slots, c,
                                                          reinterpret_cast<unsigned long long*>(c + 1),
                                                          reinterpret_cast<long long*>(peer_ready_flag), status);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

int po_p2p_recv(const float* ring, int64_t slot_elems, int32_t slots, float* dst, int64_t n, int64_t* ctl,
                const int64_t* ready_flag, int64_t* peer_ack_flag, int64_t timeout_ms, int32_t* status,
                void* stream) {
  if (n < 0 || slots < 1 || slot_elems < n || ctl == nullptr || ready_flag == nullptr || peer_ack_flag == nullptr ||
      status == nullptr || ring == nullptr || (n > 0 && dst == nullptr) || (slot_elems & 3) != 0)
    return PO_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  long long* c = reinterpret_cast<long long*>(ctl) + 2;
  p2p_wait_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const long long*>(ready_flag), c, 0, cycles(timeout_ms),
                                   status);
  p2p_copy_signal_kernel<false><<<p2p_grid(n), 256, 0, s>>>(ring, dst, n, slot_elems, slots, c,
                                                           reinterpret_cast<unsigned long long*>(c + 1),
                                                           reinterpret_cast<long long*>(peer_ack_flag), status);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"

// ---- CUDA IPC buffers ----------------------------------------------------------------------
// Buffers shared between the ranks of a node are plain cudaMalloc
// allocations (zero-filled) exported with cudaIpcGetMemHandle; a peer maps
// one with cudaIpcOpenMemHandle(cudaIpcMemLazyEnablePeerAccess) while ITS OWN
// device is current, so the mapping lives in the device that dereferences it
// and peer access (NVLink) is enabled as needed.
extern "C" {

int po_ipc_alloc(int64_t bytes, void** ptr, uint8_t* handle64) {
  if (bytes <= 0 || ptr == nullptr || handle64 == nullptr) return PO_EINVAL;
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemset(*ptr, 0, (size_t)bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return (int)e;
  }
  memcpy(handle64, &h, sizeof(h));
  return 0;
}

int po_ipc_open(const uint8_t* handle64, void** ptr) {
  if (handle64 == nullptr || ptr == nullptr) return PO_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? 0 : (int)e;
}

int po_ipc_close(void* ptr) {
  if (ptr == nullptr) return PO_EINVAL;
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? 0 : (int)e;
}

int po_ipc_free(void* ptr) {
  if (ptr == nullptr) return PO_EINVAL;
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
