// pipeoptim_pdl.cuh — programmatic dependent launch (PDL) for the short
// stream kernels (K1/K2/K3, the split-K / ReLU epilogues, the head and loss
// kernels). With po_set_pdl(1) they are launched with the programmatic
// stream-serialisation attribute: the next kernel's CTAs may be scheduled
// while this one drains, and every kernel waits (griddepcontrol.wait) for its
// predecessor's completion and memory before touching global memory — so the
// results are those of plain stream order (bit-identical runs, measured).
// Off by default. Where a stage is alone on its GPU the CUDA graphs already
// leave no launch gaps — config-1 units -0.15 us on stages 0-2, +2.5 us on
// the head stage, serial runs -1 % (profiles/r2_pdl_alone_probe.jsonl) — so
// only the stage-concurrent runner turns it on (runtime.SHARED_GPU_PDL,
// together with its shared-GPU GEMM and launch-shape policies: +2-3 %,
// profiles/r2_shared_gpu_pdl_probe.jsonl; round 1's shapes lost 2.4 % with
// it). Without the launch attribute griddepcontrol.wait is a no-op.
#pragma once

#include <cuda_runtime.h>

#include "pipeoptim.h"

namespace {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  if (!po_get_pdl()) {
    kernel<<<grid, block, smem, s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace
