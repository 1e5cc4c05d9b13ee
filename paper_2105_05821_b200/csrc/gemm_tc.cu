// Tensor-core (tcgen05) path of K2 — placeholder until the kernels land.
#include "model.cuh"

namespace simnet {
struct TcModel {};
TcModel* tc_model_create(const DevModel&, const float*, int, cudaStream_t) {
  throw ApiError("tensor-core precisions are not built yet");
}
void tc_model_destroy(TcModel* t) { delete t; }
uint64_t tc_forward(const DevModel&, int, const float*, uint32_t, uint64_t, const ForwardBuffers&,
                    cudaStream_t) {
  throw ApiError("tensor-core precisions are not built yet");
}
}  // namespace simnet
