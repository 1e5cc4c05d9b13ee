// Kernel launch with programmatic dependent launch (PDL): the kernel may start
// while its stream predecessor drains; it must execute griddepcontrol.wait
// before touching the predecessor's outputs.  Captured into CUDA graphs as
// programmatic edges.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "host_util.cuh"

namespace simnet {

// Programmatic dependent launch per launch tag.  Default: the fused round's
// front ("front") and its FC1 ("layer": f32 modes, "layer_bf16": bf16 / fp8)
// -- measured A/B on B200 at K=1024: tf32x3 35.9 -> 34.2 us per round (front +
// layer); bf16 19.8 -> 18.9 and fp8 18.2 -> 17.3 with layer_bf16 (early in the
// round it measured slower, before the FC1 epilogue became a TMA store).
// SIMNET_PDL overrides: "0" = none, "1" / "all" = every launch, else a comma
// list of tags.
inline bool pdl_enabled(const char* tag) {
  static const char* env = std::getenv("SIMNET_PDL");
  const std::string t = tag ? tag : "";
  if (!env) return t == "front" || t == "layer" || t == "layer_bf16";
  const std::string e(env);
  if (e.empty() || e == "0") return false;
  if (e == "1" || e == "all") return true;
  return !t.empty() && ("," + e + ",").find("," + t + ",") != std::string::npos;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl_tag(const char* tag, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                           cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(tag) ? 1 : 0;
  CUDA_OK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// Untagged launches (the unfused path): PDL only when SIMNET_PDL=1/all.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  launch_pdl_tag(nullptr, kernel, grid, block, smem, stream, static_cast<Args&&>(args)...);
}

}  // namespace simnet
