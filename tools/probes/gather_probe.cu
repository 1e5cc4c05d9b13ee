// Diagnostics probe: 8 warps each load 32 rows x 192 B (6 KB) with 32-B loads,
// (a) lane = row (each instruction touches 32 rows), (b) lanes over consecutive
// 32-B pieces (each instruction touches ~5 rows).  Rows are warm in L2.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gp(const float* __restrict__ stat, int mode, long long* out, float* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* base = stat + (static_cast<size_t>(blockIdx.x) * 8 + warp) * 32 * 48;
  __syncthreads();
  long long t0 = clock64();
  float acc = 0.0f;
  float w[48];
  if (mode == 0) {
    const float* row = base + lane * 48;
#pragma unroll
    for (int i = 0; i < 6; ++i)
      asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(w[8 * i]), "=f"(w[8 * i + 1]), "=f"(w[8 * i + 2]), "=f"(w[8 * i + 3]), "=f"(w[8 * i + 4]),
                     "=f"(w[8 * i + 5]), "=f"(w[8 * i + 6]), "=f"(w[8 * i + 7])
                   : "l"(row + 8 * i));
  } else {
#pragma unroll
    for (int i = 0; i < 6; ++i)
      asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(w[8 * i]), "=f"(w[8 * i + 1]), "=f"(w[8 * i + 2]), "=f"(w[8 * i + 3]), "=f"(w[8 * i + 4]),
                     "=f"(w[8 * i + 5]), "=f"(w[8 * i + 6]), "=f"(w[8 * i + 7])
                   : "l"(base + (lane + 32 * i) * 8));
  }
#pragma unroll
  for (int i = 0; i < 48; ++i) acc += w[i];
  __syncthreads();
  long long t1 = clock64();
  if (acc == 1234.5f) sink[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

extern "C" int probe(int ctas, int mode, long long* host) {
  static float* stat = nullptr;
  static float* sink = nullptr;
  const size_t n = static_cast<size_t>(ctas) * 8 * 32 * 48;
  if (!stat) {
    cudaMalloc(&stat, 148 * 8 * 32 * 48 * sizeof(float));
    cudaMalloc(&sink, 64);
    cudaMemset(stat, 0, 148 * 8 * 32 * 48 * sizeof(float));
  }
  long long* d;
  cudaMalloc(&d, ctas * sizeof(long long));
  gp<<<ctas, 256>>>(stat, mode, d, sink);  // warm
  gp<<<ctas, 256>>>(stat, mode, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, d, ctas * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  (void)n;
  return e;
}
