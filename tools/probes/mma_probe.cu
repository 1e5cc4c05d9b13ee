// Diagnostics probe: issue cost of back-to-back tcgen05.mma (one CTA, one
// thread issuing), kind::tf32 / kind::f16, M = 128, N in {64, 128, 256},
// A from shared memory (SS) or tensor memory (TS), one accumulator or
// alternating between two.  Operand contents are irrelevant (zeros).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2105_05821_b200/csrc/tc_common.cuh"

using namespace simnet;

template <int kMode>
__global__ void mma_probe(int n, int count, int ts, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (nacc >= 10 && threadIdx.x < 32) {  // warp-wide issue: uniform operands, elect.sync picks the issuing lane
    nacc -= 10;
    const uint32_t idesc = instr_desc(kMode == kBF16 ? 1 : 2, n);
    const uint64_t ad = smem_desc_sw128(su32(base));
    const uint64_t bd = smem_desc_sw128(su32(base + 32 * 1024));
    long long t0 = clock64();
    for (int i = 0; i < count; ++i) {
      const uint32_t d = tmem + (nacc > 1 ? (i & 1) * n : 0);
      const uint32_t acc = i > 1;
      if (ts) {
        const uint32_t a = tmem + 448 + (i & 3) * 8;
        asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(bd),
                     "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad + ((i & 3) * 2)),
                     "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      long long t2 = clock64();
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
    __syncwarp();
  } else if (threadIdx.x == 0) {
    const uint32_t idesc = instr_desc(kMode == kBF16 ? 1 : 2, n);
    const uint64_t ad = smem_desc_sw128(su32(base));
    const uint64_t bd = smem_desc_sw128(su32(base + 32 * 1024));
    long long t0 = clock64();
    for (int i = 0; i < count; ++i) {
      const uint32_t d = tmem + (nacc > 1 ? (i & 1) * n : 0);
      if (ts)
        mma_ts<kMode>(d, tmem + 512 - 32 + (i & 3) * 8 - 32, bd, idesc, i > 1);
      else
        mma<kMode>(d, ad + ((i & 3) * 2), bd, idesc, i > 1);
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// 3xTF32 k-step patterns, N = n output channels (SS):
//   pattern 0: Alo*Whi, Ahi*Wlo, Ahi*Whi into one accumulator (3 MMAs of N)
//   pattern 1: Ahi*[Whi;Wlo] (one MMA of 2N) + Alo*Whi into the cross half (N)
__global__ void ksteps_probe(int n, int ksteps, int pattern, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t id1 = instr_desc(2, n), id2 = instr_desc(2, 2 * n);
    const uint32_t ahi = su32(base), alo = su32(base + 16384), whi = su32(base + 32768), wlo = whi + n * 128;
    long long t0 = clock64();
    for (int s = 0; s < ksteps; ++s) {
      const int j = s & 3;
      const uint64_t dah = smem_desc_sw128(ahi + j * 32), dal = smem_desc_sw128(alo + j * 32);
      const uint64_t dwh = smem_desc_sw128(whi + j * 32), dwl = smem_desc_sw128(wlo + j * 32);
      if (pattern == 0) {
        mma<kTF32>(tmem, dal, dwh, id1, s > 0);
        mma<kTF32>(tmem, dah, dwl, id1, 1);
        mma<kTF32>(tmem, dah, dwh, id1, 1);
      } else {
        mma<kTF32>(tmem, dah, dwh, id2, s > 0);       // [main | cross] = Ahi * [Whi ; Wlo]
        mma<kTF32>(tmem + n, dal, dwh, id1, 1);       // cross += Alo * Whi
      }
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

extern "C" int probe_ksteps(int n, int ksteps, int pattern, long long* host) {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  const size_t sm = 100 * 1024;
  cudaFuncSetAttribute(ksteps_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  ksteps_probe<<<1, 128, sm>>>(n, ksteps, pattern, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

extern "C" int probe(int mode, int n, int count, int ts, int nacc, long long* host) {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  const size_t sm = 100 * 1024;
  if (mode == kBF16) {
    cudaFuncSetAttribute(mma_probe<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    mma_probe<kBF16><<<1, 128, sm>>>(n, count, ts, nacc, d);
  } else {
    cudaFuncSetAttribute(mma_probe<kTF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    mma_probe<kTF32><<<1, 128, sm>>>(n, count, ts, nacc, d);
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}
