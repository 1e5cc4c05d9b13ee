// K2 (latency-predictor inference) layer GEMM interfaces.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace simnet {

// One CNN layer as a GEMM over (sample, position) rows: the k2/s2 window of
// output position p is input rows 2p, 2p+1 laid end to end, so every layer's
// input is the previous output viewed as [rows/2 x 2*channels] (cnn.cpp:97-98).
struct LayerGemm {
  const float* a;          // input activations
  uint64_t m;              // output rows = samples * rows_per_sample
  int rows_per_sample;     // output positions per sample
  int valid_rows;          // rows stored per sample; rows >= valid_rows read as 0
  int kdim;                // 2 * input channels (or flat dim for FC)
  uint64_t sample_stride;  // floats between samples in `a`
  const float* w;          // [kdim][n], n contiguous (reference column-major)
  const float* w2;         // residual projection, same layout (or null)
  const float* bias;       // [n]
  float* c;                // [m][ldc]
  int n, ldc;
  int relu;
  float* splitk;           // scratch for the small-batch split-K path ([m][chunks][n] floats), or null
  int chunk;               // accumulation order: 0 = one fma chain over all of K (k ascending);
                           // kSgemmChunk = chains over 512-wide K chunks, summed in chunk order
};

// Accumulation order.  chunk == 0: one fma chain per output, k ascending from
// 0 -- the reference's restated forward (oracle/cnn_restated.cpp gemm_cm, cnn.cpp
// column-major order), used for every layer of the CNN models.  chunk ==
// kSgemmChunk: each 512-wide chunk's fma chain starts at 0 (k ascending) and
// the chunk sums are added in order -- the FC-only predictor's definition (no
// reference implementation; the oracle port defines it the same way), which
// lets its 5550-wide FC1 split over K.  Every batch size and both kernels below
// use the layer's order, so results stay batch-independent.
constexpr int kSgemmChunk = 512;
constexpr uint64_t kSgemvMaxM = 8;  // batches up to this many rows take the split-K GEMV
inline uint64_t sgemm_splitk_floats(uint64_t m, int kdim, int n) {
  return m * static_cast<uint64_t>((kdim + kSgemmChunk - 1) / kSgemmChunk) * static_cast<uint64_t>(n);
}

void launch_sgemm(const LayerGemm& g, cudaStream_t stream);
bool sgemm_two_launches(const LayerGemm& g);  // the split-K GEMV path (2 kernels)

}  // namespace simnet
