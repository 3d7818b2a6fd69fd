// nvls_probe.cu — does this box support NVLink SHARP multicast objects
// (cuMulticast*) and multimem.ld_reduce? One device, one process: creates a
// 1-device multicast object, binds a physical allocation, maps the multicast
// address and reads it back through multimem.ld_reduce.add.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o gpurun_out/nvls_probe scripts/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#define CK(x)                                                                \
  do {                                                                       \
    CUresult r_ = (x);                                                       \
    if (r_ != CUDA_SUCCESS) {                                                \
      const char* s_ = nullptr;                                              \
      cuGetErrorString(r_, &s_);                                             \
      printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?");              \
      return 1;                                                              \
    }                                                                        \
  } while (0)

__global__ void ld_reduce(const float* mc, float* out, int n4) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float a, b, c, d;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
               : "l"(mc + 4 * i)
               : "memory");
  out[4 * i] = a;
  out[4 * i + 1] = b;
  out[4 * i + 2] = c;
  out[4 * i + 3] = d;
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mc = 0, fabric = 0, posix = 0;
  cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handles=%d posix_fd_handles=%d\n", mc, fabric, posix);
  cudaSetDevice(0);
  CUcontext ctx;
  CK(cuCtxGetCurrent(&ctx));
  if (!mc) return 0;
  const size_t n = 1 << 20, bytes = n * sizeof(float);
  CUmulticastObjectProp prop = {};
  prop.numDevices = 1;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop.size = bytes;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  prop.size = (bytes + gran - 1) / gran * gran;
  printf("multicast granularity %zu, size %zu\n", gran, prop.size);
  CUmemGenericAllocationHandle mch;
  // creation matrix: devices x handle types x granularity kind
  for (int nd = 1; nd <= 2; ++nd)
    for (int gk = 0; gk < 2; ++gk)
      for (int t : {0, 1, 8}) {
        CUmulticastObjectProp p3 = {};
        p3.numDevices = nd;
        p3.handleTypes = (unsigned long long)t;
        p3.size = 1 << 21;
        size_t g3 = 0;
        CUresult rg = cuMulticastGetGranularity(&g3, &p3, gk ? CU_MULTICAST_GRANULARITY_RECOMMENDED
                                                             : CU_MULTICAST_GRANULARITY_MINIMUM);
        if (rg == CUDA_SUCCESS && g3) p3.size = (p3.size + g3 - 1) / g3 * g3;
        CUmemGenericAllocationHandle h3;
        CUresult r3 = cuMulticastCreate(&h3, &p3);
        const char* es = nullptr;
        cuGetErrorString(r3, &es);
        printf("matrix numDevices=%d gran=%s(%zu, rc %d) handleTypes=%d size=%zu -> %d %s\n", nd,
               gk ? "recommended" : "minimum", g3, (int)rg, t, p3.size, (int)r3, es ? es : "?");
        if (r3 == CUDA_SUCCESS) cuMemRelease(h3);
      }
  // which handle types does cuMulticastCreate accept with one device?
  const int types[3] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
  int ok_type = -1;
  for (int t : types) {
    CUmulticastObjectProp p2 = prop;
    p2.handleTypes = (unsigned long long)t;
    CUresult r = cuMulticastCreate(&mch, &p2);
    const char* es = nullptr;
    cuGetErrorString(r, &es);
    printf("cuMulticastCreate(numDevices=1, handleTypes=%d) -> %d %s\n", t, (int)r, es ? es : "?");
    if (r == CUDA_SUCCESS && ok_type < 0) {
      ok_type = t;
      break;
    }
  }
  if (ok_type < 0) return 0;
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle ph;
  CK(cuMemCreate(&ph, prop.size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, ph, 0, prop.size, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0));
  CK(cuMemMap(uc, prop.size, 0, ph, 0));
  CK(cuMemAddressReserve(&mcp, prop.size, gran, 0, 0));
  CK(cuMemMap(mcp, prop.size, 0, mch, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, prop.size, &acc, 1));
  CK(cuMemSetAccess(mcp, prop.size, &acc, 1));
  float* h = new float[n];
  for (size_t i = 0; i < n; ++i) h[i] = 0.5f * (float)(i % 1000);
  cudaMemcpy((void*)uc, h, bytes, cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, bytes);
  ld_reduce<<<(n / 4 + 255) / 256, 256>>>((const float*)mcp, out, (int)(n / 4));
  cudaError_t e = cudaDeviceSynchronize();
  printf("ld_reduce kernel: %s\n", cudaGetErrorString(e));
  float* r = new float[n];
  cudaMemcpy(r, out, bytes, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) bad += r[i] != h[i];
  printf("mismatches %zu of %zu (1-device multicast sum == the buffer)\n", bad, n);
  return 0;
}
