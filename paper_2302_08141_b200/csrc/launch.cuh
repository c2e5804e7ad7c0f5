// launch.cuh — programmatic dependent launch (PDL) for the compute kernels.
//
// Inside a step list, a GEMM / elementwise kernel that follows another compute kernel on the
// same stream is launched with cudaLaunchAttributeProgrammaticStreamSerialization (the executor
// sets PdlEnabled() per step, abi.cpp RunOnce): its CTAs may be scheduled while the previous
// kernel drains, run their prologue (barrier init, TMEM alloc, tensor-map prefetch, table
// staging) and then block in griddepcontrol.wait until the previous grid has completed and its
// writes are visible.  Every kernel launched through LaunchPdl calls PdlTrigger() early and
// PdlWait() before its first read of a predecessor's output; without the attribute both are
// no-ops.  Kernels that spin on peers (the resharding pulls) are never launched this way and a
// kernel after them never gets the attribute, so a waiting CTA can only wait for a grid that
// makes progress on its own.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "kernels.h"
#include "pdl.cuh"

namespace rh {

template <typename... KArgs, typename... Args>
inline void LaunchPdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                      Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  if (PdlEnabled()) {
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  RH_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace rh
