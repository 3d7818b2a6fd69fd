// pipeoptim_nvls.cu — NVLink SHARP (NVLS) multicast objects for the sharded
// hybrid-DP update (po_step_predict_dp_shard with a po_dp_multicast).
//
// One multicast object per DP group spans all of a replica's update buffers
// (both gradient parities, W, state, W_hat). The creating replica exports it
// as a POSIX file descriptor (passed to the others over a UNIX socket by the
// host, dp_fused.py); every replica imports it, adds its device, and binds
// ONE local physical allocation of the object's size to it. The replica then
// holds a unicast VA of its own copy (its buffers) and a multicast VA: a
// multimem.ld_reduce through the multicast VA returns the sum over all
// replicas' copies computed in the NVSwitch, a multimem.st writes every copy.
//
// Driver-API errors are returned as PO_EDRIVER_BASE + CUresult.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <unistd.h>

#include "pipeoptim.h"

struct po_nvls {
  CUmemGenericAllocationHandle mc = 0;    // the multicast object
  CUmemGenericAllocationHandle phys = 0;  // this replica's physical memory
  CUdeviceptr uc = 0, mc_va = 0;
  size_t size = 0, gran = 0;
  int n_devices = 0;
  bool added = false, bound = false, mapped_uc = false, mapped_mc = false;
};

namespace {

// Driver entry points are resolved at run time through the runtime
// (cudaGetDriverEntryPoint): the library keeps no link-time dependency on
// libcuda, so it still loads (for the ABI checks) where no driver exists.
template <typename F>
F entry(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}

#define PO_DRIVER_FUNCS(X)                                                                        \
  X(cuDeviceGet) X(cuDeviceGetAttribute) X(cuMulticastGetGranularity) X(cuMulticastCreate)           \
  X(cuMemRelease) X(cuMemExportToShareableHandle) X(cuMemImportFromShareableHandle)                   \
  X(cuMulticastAddDevice) X(cuMemCreate) X(cuMulticastBindMem) X(cuMemAddressReserve) X(cuMemMap)     \
  X(cuMemSetAccess) X(cuMemsetD8) X(cuCtxSynchronize) X(cuMemUnmap) X(cuMemAddressFree)               \
  X(cuMulticastUnbind)

struct Driver {
#define PO_DECL(f) decltype(&::f) p_##f = nullptr;
  PO_DRIVER_FUNCS(PO_DECL)
#undef PO_DECL
  bool ok = true;
};

// every entry point, resolved once (ok = false if any is missing)
const Driver& api() {
  static const Driver d = [] {
    Driver r;
#define PO_LOAD(f)                          \
  r.p_##f = entry<decltype(&::f)>(#f);      \
  r.ok = r.ok && r.p_##f != nullptr;
    PO_DRIVER_FUNCS(PO_LOAD)
#undef PO_LOAD
    return r;
  }();
  return d;
}

int drv(CUresult r) { return r == CUDA_SUCCESS ? 0 : PO_EDRIVER_BASE + (int)r; }

int current_device(CUdevice* dev) {
  if (!api().ok) return PO_EDRIVER_BASE + (int)CUDA_ERROR_NOT_FOUND;  // driver lacks an entry point
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return (int)e;
  cudaFree(nullptr);  // make sure the primary context exists
  return drv(api().p_cuDeviceGet(dev, d));
}

CUmulticastObjectProp props(int n_devices, size_t size) {
  CUmulticastObjectProp p = {};
  p.numDevices = (unsigned)n_devices;
  p.size = size;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

int granularity(int n_devices, size_t bytes, size_t* gran) {
  CUmulticastObjectProp p = props(n_devices, bytes);
  return drv(api().p_cuMulticastGetGranularity(gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED));
}

}  // namespace

extern "C" {

int po_nvls_probe(int32_t n_devices, int64_t bytes, int64_t* granularity_out) {
  if (n_devices < 1 || bytes <= 0) return PO_EINVAL;
  CUdevice dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  int supported = 0;
  rc = drv(api().p_cuDeviceGetAttribute(&supported, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  if (rc) return rc;
  if (!supported) return PO_EDRIVER_BASE + (int)CUDA_ERROR_NOT_SUPPORTED;
  size_t gran = 0;
  rc = granularity(n_devices, (size_t)bytes, &gran);
  if (rc) return rc;
  if (granularity_out) *granularity_out = (int64_t)gran;
  CUmulticastObjectProp p = props(n_devices, ((size_t)bytes + gran - 1) / gran * gran);
  CUmemGenericAllocationHandle h;
  rc = drv(api().p_cuMulticastCreate(&h, &p));
  if (rc) return rc;
  return drv(api().p_cuMemRelease(h));
}

int po_nvls_create(int32_t n_devices, int64_t bytes, int32_t* fd_out, po_nvls** out) {
  if (n_devices < 1 || bytes <= 0 || fd_out == nullptr || out == nullptr) return PO_EINVAL;
  CUdevice dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  po_nvls* g = new po_nvls();
  g->n_devices = n_devices;
  rc = granularity(n_devices, (size_t)bytes, &g->gran);
  if (!rc) {
    g->size = ((size_t)bytes + g->gran - 1) / g->gran * g->gran;
    CUmulticastObjectProp p = props(n_devices, g->size);
    rc = drv(api().p_cuMulticastCreate(&g->mc, &p));
  }
  int fd = -1;
  if (!rc) rc = drv(api().p_cuMemExportToShareableHandle(&fd, g->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  if (rc) {
    if (g->mc) api().p_cuMemRelease(g->mc);
    delete g;
    return rc;
  }
  *fd_out = fd;
  *out = g;
  return 0;
}

int po_nvls_open(int32_t fd, int32_t n_devices, int64_t bytes, po_nvls** out) {
  if (fd < 0 || n_devices < 1 || bytes <= 0 || out == nullptr) return PO_EINVAL;
  CUdevice dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  po_nvls* g = new po_nvls();
  g->n_devices = n_devices;
  rc = granularity(n_devices, (size_t)bytes, &g->gran);
  if (!rc) {
    g->size = ((size_t)bytes + g->gran - 1) / g->gran * g->gran;
    rc = drv(api().p_cuMemImportFromShareableHandle(&g->mc, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  }
  if (rc) {
    delete g;
    return rc;
  }
  *out = g;
  return 0;
}

// Every replica, before any replica binds memory.
int po_nvls_add_device(po_nvls* g) {
  if (g == nullptr || g->added) return PO_EINVAL;
  CUdevice dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  rc = drv(api().p_cuMulticastAddDevice(g->mc, dev));
  if (!rc) g->added = true;
  return rc;
}

// After every replica added its device: this replica's physical memory
// (zero-filled), bound to the object, mapped at a unicast and a multicast VA.
int po_nvls_bind(po_nvls* g, void** uc_ptr, void** mc_ptr) {
  if (g == nullptr || !g->added || g->bound || uc_ptr == nullptr || mc_ptr == nullptr) return PO_EINVAL;
  CUdevice dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = (int)dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  rc = drv(api().p_cuMemCreate(&g->phys, g->size, &ap, 0));
  if (rc) return rc;
  rc = drv(api().p_cuMulticastBindMem(g->mc, 0, g->phys, 0, g->size, 0));
  if (rc) return rc;
  g->bound = true;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = (int)dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  rc = drv(api().p_cuMemAddressReserve(&g->uc, g->size, g->gran, 0, 0));
  if (!rc) rc = drv(api().p_cuMemMap(g->uc, g->size, 0, g->phys, 0));
  if (!rc) g->mapped_uc = true;
  if (!rc) rc = drv(api().p_cuMemSetAccess(g->uc, g->size, &acc, 1));
  if (!rc) rc = drv(api().p_cuMemAddressReserve(&g->mc_va, g->size, g->gran, 0, 0));
  if (!rc) rc = drv(api().p_cuMemMap(g->mc_va, g->size, 0, g->mc, 0));
  if (!rc) g->mapped_mc = true;
  if (!rc) rc = drv(api().p_cuMemSetAccess(g->mc_va, g->size, &acc, 1));
  if (!rc) rc = drv(api().p_cuMemsetD8(g->uc, 0, g->size));
  if (!rc) rc = drv(api().p_cuCtxSynchronize());
  if (rc) return rc;
  *uc_ptr = (void*)g->uc;
  *mc_ptr = (void*)g->mc_va;
  return 0;
}

int64_t po_nvls_size(const po_nvls* g) { return g == nullptr ? 0 : (int64_t)g->size; }

int po_nvls_free(po_nvls* g) {
  if (g == nullptr) return PO_EINVAL;
  api().p_cuCtxSynchronize();
  if (g->mapped_mc) api().p_cuMemUnmap(g->mc_va, g->size);
  if (g->mc_va) api().p_cuMemAddressFree(g->mc_va, g->size);
  if (g->mapped_uc) api().p_cuMemUnmap(g->uc, g->size);
  if (g->uc) api().p_cuMemAddressFree(g->uc, g->size);
  if (g->bound) {
    CUdevice dev;
    if (current_device(&dev) == 0) api().p_cuMulticastUnbind(g->mc, dev, 0, g->size);
  }
  if (g->phys) api().p_cuMemRelease(g->phys);
  if (g->mc) api().p_cuMemRelease(g->mc);
  delete g;
  return 0;
}

}  // extern "C"
