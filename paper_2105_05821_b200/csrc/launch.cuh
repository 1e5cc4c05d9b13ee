// Kernel launch with programmatic dependent launch (PDL): the kernel may start
// while its stream predecessor drains; it must execute griddepcontrol.wait
// before touching the predecessor's outputs.  Captured into CUDA graphs as
// programmatic edges.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include "host_util.cuh"

namespace simnet {

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // Opt-in: measured slower on B200 for this round loop (early dependents
  // launch and then contend with the running kernel), so off by default.
  static const bool disabled = std::getenv("SIMNET_PDL") == nullptr;
  cfg.attrs = attr;
  cfg.numAttrs = disabled ? 0 : 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

}  // namespace simnet
