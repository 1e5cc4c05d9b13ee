// Diagnostics probe: per-CTA arrival times of four 16 KB bulk copies (issued
// together) from a buffer that was (a) just written by another kernel,
// (b) read before (warm), (c) never touched since allocation.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void writer(float4* buf, size_t n4, float v) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
    buf[i] = make_float4(v, v, v, v);
}

__global__ void reader(const uint8_t* src, long long* out, int nchunks, int chunk_bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < nchunks; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int i = 0; i < nchunks; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[i])), "r"(chunk_bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(sm + i * chunk_bytes)),
                   "l"(src + (static_cast<size_t>(blockIdx.x) * nchunks + i) * chunk_bytes), "r"(chunk_bytes),
                   "r"(su32(&bar[i]))
                   : "memory");
    }
    for (int i = 0; i < nchunks; ++i) {
      uint32_t ok = 0;
      do {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(su32(&bar[i])) : "memory");
      } while (!ok);
      out[blockIdx.x * 8 + i] = clock64() - t0;
    }
  }
}

extern "C" int probe(int ctas, int nchunks, int chunk_bytes, int mode, long long* host_out) {
  size_t bytes = static_cast<size_t>(ctas) * nchunks * chunk_bytes;
  static uint8_t* buf = nullptr;
  static size_t cap = 0;
  if (cap < bytes) {
    if (buf) cudaFree(buf);
    cudaMalloc(&buf, bytes);
    cap = bytes;
  }
  long long* d_out;
  cudaMalloc(&d_out, ctas * 8 * sizeof(long long));
  cudaFuncSetAttribute(reader, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (mode == 0) writer<<<148, 512>>>(reinterpret_cast<float4*>(buf), bytes / 16, 1.0f);      // just written
  if (mode == 1) reader<<<ctas, 32, nchunks * chunk_bytes>>>(buf, d_out, nchunks, chunk_bytes);  // warm read first
  if (mode == 2) {  // flush L2 by writing a large other buffer
    static uint8_t* big = nullptr;
    if (!big) cudaMalloc(&big, 512ull << 20);
    writer<<<148 * 4, 512>>>(reinterpret_cast<float4*>(big), (512ull << 20) / 16, 2.0f);
  }
  reader<<<ctas, 32, nchunks * chunk_bytes>>>(buf, d_out, nchunks, chunk_bytes);
  cudaMemcpy(host_out, d_out, ctas * 8 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  return cudaGetLastError();
}
