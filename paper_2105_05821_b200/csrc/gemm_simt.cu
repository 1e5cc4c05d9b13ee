// FP32 SIMT path of K2 (precision ILSIM_PREC_FP32): one tiled FFMA GEMM per
// layer, C = act(A * W + b) with the reference's parameter layout
// (column-major W[o + k*rows] == [K x N] N-contiguous, cnn.cpp:99-124).
// The fp32 correctness anchor for the tensor-core paths; products are exact
// fp32 FMAs accumulated k-ascending per output, then bias, then ReLU.
#include "gemm.cuh"

namespace simnet {

namespace {
constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256) sgemm_kernel(LayerGemm g) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const uint64_t row0 = static_cast<uint64_t>(blockIdx.x) * BM;
  const int col0 = blockIdx.y * BN;

  // A-tile loader: row (tid / 4), k chunk (tid % 4) * 4
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  const uint64_t gr = row0 + lr;
  const float* arow = nullptr;
  if (gr < g.m) {
    const uint64_t sidx = gr / g.rows_per_sample;
    const int pidx = static_cast<int>(gr - sidx * g.rows_per_sample);
    if (pidx < g.valid_rows) arow = g.a + sidx * g.sample_stride + static_cast<uint64_t>(pidx) * g.kdim;
  }
  // B-tile loader: k (tid / 16), n chunk (tid % 16) * 4
  const int bk = tid >> 4, bn = (tid & 15) * 4;

  // Residual layers (cnn.cpp:104-107; oracle/cnn_restated.cpp): the W chain,
  // then the P chain continuing on the same accumulator (the reference adds
  // P * in into the W product before the bias), i.e. two passes over K.
  float acc[4][4] = {};
  float tot[4][4] = {};  // sum of the finished kSgemmChunk chunks (see gemm.cuh)
  const int passes = g.w2 ? 2 : 1;
  for (int pass = 0; pass < passes; ++pass) {
    const float* wsrc = pass == 0 ? g.w : g.w2;
    for (int k0 = 0; k0 < g.kdim; k0 += BK) {
      if (g.chunk > 0 && (pass > 0 || k0 > 0) && k0 % g.chunk == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            tot[i][j] += acc[i][j];
            acc[i][j] = 0.0f;
          }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int k = k0 + lk + t;
        As[lk + t][lr] = (arow && k < g.kdim) ? arow[k] : 0.0f;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int k = k0 + bk, n = col0 + bn + t;
        const bool ok = k < g.kdim && n < g.n;
        Bs[bk][bn + t] = ok ? wsrc[static_cast<uint64_t>(k) * g.n + n] : 0.0f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t r = row0 + ty + 16 * i;
    if (r >= g.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = col0 + tx + 16 * j;
      if (n >= g.n) continue;
      float v = tot[i][j] + acc[i][j];
      v += g.bias[n];
      if (g.relu) v = fmaxf(v, 0.0f);
      g.c[r * g.ldc + n] = v;
    }
  }
}
// Small batches (the sequential / FC-only configurations): one thread per
// (row, output), one CTA per (128 outputs, K chunk, row); the chunk's fma
// chain as in sgemm_kernel, written to the scratch, then summed in chunk order.
constexpr int kGv = 128;
__global__ void __launch_bounds__(kGv) sgemv_chunk_kernel(LayerGemm g) {
  __shared__ float as[kSgemmChunk];
  const int n = blockIdx.x * kGv + threadIdx.x;
  const int c = blockIdx.y;
  const uint64_t r = blockIdx.z;
  const int k0 = c * kSgemmChunk, k1 = min(g.kdim, k0 + kSgemmChunk);
  const float* arow = g.a + r * g.sample_stride;
  for (int k = k0 + threadIdx.x; k < k1; k += kGv) as[k - k0] = arow[k];
  __syncthreads();
  if (n >= g.n) return;
  const float* w = g.w + static_cast<uint64_t>(k0) * g.n + n;
  float acc = 0.0f;
  int k = k0;
#pragma unroll 8
  for (; k < k1; ++k, w += g.n) acc = fmaf(as[k - k0], __ldg(w), acc);
  const int chunks = gridDim.y;
  g.splitk[(r * chunks + c) * g.n + n] = acc;
}

__global__ void __launch_bounds__(kGv) sgemv_reduce_kernel(LayerGemm g, int chunks) {
  const int n = blockIdx.x * kGv + threadIdx.x;
  const uint64_t r = blockIdx.y;
  if (n >= g.n) return;
  float tot = 0.0f;
  for (int c = 0; c < chunks; ++c) tot += g.splitk[(r * chunks + c) * g.n + n];
  float v = tot + g.bias[n];
  if (g.relu) v = fmaxf(v, 0.0f);
  g.c[r * g.ldc + n] = v;
}
}  // namespace

void launch_sgemm(const LayerGemm& g, cudaStream_t stream) {
  if (g.m == 0) return;
  if (sgemm_two_launches(g)) {
    const int chunks = (g.kdim + kSgemmChunk - 1) / kSgemmChunk;
    const unsigned gx = static_cast<unsigned>((g.n + kGv - 1) / kGv);
    sgemv_chunk_kernel<<<dim3(gx, chunks, static_cast<unsigned>(g.m)), kGv, 0, stream>>>(g);
    sgemv_reduce_kernel<<<dim3(gx, static_cast<unsigned>(g.m)), kGv, 0, stream>>>(g, chunks);
    return;
  }
  dim3 grid(static_cast<unsigned>((g.m + BM - 1) / BM), (g.n + BN - 1) / BN);
  sgemm_kernel<<<grid, 256, 0, stream>>>(g);
}

bool sgemm_two_launches(const LayerGemm& g) {
  return g.splitk && g.chunk == kSgemmChunk && g.m <= kSgemvMaxM && g.rows_per_sample == 1 && g.valid_rows == 1 &&
         !g.w2 && g.kdim > kSgemmChunk;
}

}  // namespace simnet
