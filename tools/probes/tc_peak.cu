// Tensor-core peak probe (roofline denominators).
//
// 1. issue cost: cycles per back-to-back tcgen05.mma in ONE CTA (one issuing
//    thread), M = 128, kind::{tf32, f16 (bf16), f8f6f4 (e4m3)}, N in {64, 128,
//    256}, into 1, 2 or 4 accumulators round-robin (dependency vs throughput).
// 2. dense peak: every SM runs one CTA issuing M=128 N=256 MMAs round-robin
//    over 2 accumulators with operands from shared memory filled with finite
//    pseudo-random values; FLOP/s = 2*M*N*K*count*CTAs / event time.  The
//    burst figure is one ~2 ms launch; the sustained one is ~1 s of
//    back-to-back launches (clocks under power / thermal load).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2105_05821_b200/csrc/tc_common.cuh"

using namespace simnet;

// K per MMA instruction: 32 bytes of K for every kind (tf32 8, f16 16, f8 32)
__host__ __device__ constexpr int k_of(int mode) { return mode == kFP8 ? 32 : (mode == kBF16 ? 16 : 8); }

template <int kMode>
__device__ __forceinline__ void setup(uint8_t* base, uint64_t* bar, uint32_t* slot) {
  // finite pseudo-random operand bits: sign/exponent kept small so nothing overflows
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (i * 2654435761u) ^ (blockIdx.x * 40503u);
    x ^= x >> 13;
    uint32_t v;
    if (kMode == kFP8) v = x & 0x3b3b3b3bu;          // e4m3 values |v| < 1
    else if (kMode == kBF16) v = (x & 0x807f807fu) | 0x3f003f00u;  // bf16 in [0.5, 1)
    else v = (x & 0x807fffffu) | 0x3f000000u;        // f32 in [0.5, 1)
    reinterpret_cast<uint32_t*>(base)[i] = v;
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

__device__ __forceinline__ void teardown(uint32_t tmem) {
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

template <int kMode>
__global__ void mma_loop(int n, int count, int nacc, long long* out, int a_tmem = 0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  setup<kMode>(base, &bar, &slot);
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = instr_desc(mode_fmt(kMode), n);
    const uint64_t ad = smem_desc_sw128(su32(base));
    const uint64_t bd = smem_desc_sw128(su32(base + 32 * 1024));
    const int stride = n <= 128 ? 128 : 256;  // accumulator column spacing (nacc * stride <= 512)
    long long t0 = clock64();
    for (int i = 0; i < count; ++i) {
      const uint32_t d = tmem + (i & (nacc - 1)) * stride;  // nacc: 1, 2 or 4
      if (a_tmem)  // A from tensor memory (columns 384+, left as allocated)
        mma_ts<kMode>(d, tmem + 384 + (i & 3) * 8, bd, idesc, i >= nacc);
      else
        mma<kMode>(d, ad + ((i & 3) * 2), bd, idesc, i >= nacc);
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (out && blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  teardown(tmem);
}

// The same loop issued by a whole warp with elect.sync inside the asm (the
// issuing thread chosen per instruction), instead of one thread under
// `if (threadIdx.x == 0)`: ptxas then needs no per-MMA waterfall loop
// (ELECT / BRA.U.ANY) around UTCHMMA.
__device__ __forceinline__ void mma_tf32_elect(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts_tf32_elect(uint32_t tmem, uint32_t a, uint64_t bd, uint32_t idesc,
                                                  uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
      "r"(a), "l"(bd), "r"(idesc), "r"(acc));
}
template <bool kTs>
__global__ void mma_loop_warp(int n, int count, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  setup<kTF32>(base, &bar, &slot);
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint32_t idesc = instr_desc(mode_fmt(kTF32), n);
    const uint64_t ad = smem_desc_sw128(su32(base));
    const uint64_t bd = smem_desc_sw128(su32(base + 32 * 1024));
    const int stride = n <= 128 ? 128 : 256;
    long long t0 = clock64();
    for (int i = 0; i < count; ++i) {
      const uint32_t d = tmem + (i & (nacc - 1)) * stride;
      if constexpr (kTs)
        mma_ts_tf32_elect(d, tmem + 384 + (i & 3) * 8, bd, idesc, i >= nacc);
      else
        mma_tf32_elect(d, ad + ((i & 3) * 2), bd, idesc, i >= nacc);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
    __syncwarp();
    long long t2 = clock64();
    if (out && blockIdx.x == 0 && threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  teardown(tmem);
}
extern "C" int issue_cost_warp(int n, int count, int nacc, long long* host, int ts) {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  const size_t sm = 100 * 1024;
  if (ts) {
    cudaFuncSetAttribute(mma_loop_warp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    mma_loop_warp<true><<<1, 128, sm>>>(n, count, nacc, d);
  } else {
    cudaFuncSetAttribute(mma_loop_warp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    mma_loop_warp<false><<<1, 128, sm>>>(n, count, nacc, d);
  }
  int e = cudaGetLastError();
  if (!e) e = cudaDeviceSynchronize();
  cudaMemcpy(host, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

template <int kMode>
static int launch(int grid, int n, int count, int nacc, long long* d, int a_tmem = 0) {
  const size_t sm = 100 * 1024;
  cudaFuncSetAttribute(mma_loop<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  mma_loop<kMode><<<grid, 128, sm>>>(n, count, nacc, d, a_tmem);
  return cudaGetLastError();
}

static int launch_mode(int mode, int grid, int n, int count, int nacc, long long* d) {
  if (mode == kFP8) return launch<kFP8>(grid, n, count, nacc, d);
  if (mode == kBF16) return launch<kBF16>(grid, n, count, nacc, d);
  return launch<kTF32>(grid, n, count, nacc, d);
}

// cycles (issue, complete) of `count` MMAs in one CTA
extern "C" int issue_cost(int mode, int n, int count, int nacc, long long* host) {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  int e = launch_mode(mode, 1, n, count, nacc, d);
  if (!e) e = cudaDeviceSynchronize();
  cudaMemcpy(host, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

// the same with A read from tensor memory (tcgen05.mma [d], [a_tmem], b_desc): FC1's form
extern "C" int issue_cost_ts(int mode, int n, int count, int nacc, long long* host) {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  int e = mode == kBF16 ? launch<kBF16>(1, n, count, nacc, d, 1) : launch<kTF32>(1, n, count, nacc, d, 1);
  if (!e) e = cudaDeviceSynchronize();
  cudaMemcpy(host, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

// dense TFLOP/s over `launches` back-to-back launches of `grid` CTAs x `count` MMAs
extern "C" int dense_peak(int mode, int grid, int count, int launches, double* tflops, double* ms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int e = launch_mode(mode, grid, 256, count, 2, nullptr);  // warm-up
  if (!e) e = cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < launches && !e; ++i) e = launch_mode(mode, grid, 256, count, 2, nullptr);
  cudaEventRecord(b);
  if (!e) e = cudaEventSynchronize(b);
  float t = 0;
  cudaEventElapsedTime(&t, a, b);
  const double flop = 2.0 * 128 * 256 * k_of(mode) * static_cast<double>(count) * grid * launches;
  *tflops = flop / (t * 1e-3) / 1e12;
  *ms = t;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return e;
}
