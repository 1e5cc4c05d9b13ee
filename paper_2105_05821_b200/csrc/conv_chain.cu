// K2, fused conv chain: conv0 -> conv1 -> conv2 of the C3 latency predictor
// (cnn.cpp:90-110 for each conv layer) for 8 samples per work item, entirely
// on chip.  Accumulators live in TMEM; between layers the epilogue warps read
// them (tcgen05.ld), apply bias + ReLU, and restage them in shared memory as
// the next layer's K-major SWIZZLE_128B A operand (row pairs concatenated: a
// kernel-2/stride-2 window is two adjacent rows).  Only the final conv2
// activations ("flat", 4 KB per sample) leave the SM.
//
//   TMEM (f32 columns): conv0 4 tiles x 64 [0,256) | conv1 2 x 64 [256,384) |
//                       conv2 64 [384,448);
//   3xTF32: every tile's accumulator is 128 columns [Ahi.Whi | Ahi.Wlo + Alo.Whi]
//   (the round front's stacked k-step, round_front.cu): conv0 t at 128t,
//   conv1 u at 128u, conv2 at 256 (conv0 of the next item waits for the
//   conv2 drain)
//   SMEM: R1 128 KB  = conv0 input ring (4 stages of 16 KB chunk (+16 KB lo))
//                      or the restaged A tile of conv1 / conv2
//         R2  64 KB  = the current layer's weights (hi + lo), TMA-loaded
//
//   warp 0      TMA producer (weights per layer, gathered-input chunks)
//   warp 1      TMEM allocator + tcgen05.mma issuer
//   warps 2-5   spare (K1 writes the 3xTF32 hi/lo input planes)
//   warps 6-9   epilogue: TMEM -> bias/ReLU -> restage (or -> global)
#include <cuda.h>
#include <cuda_bf16.h>

#include "conv_chain.cuh"
#include "tc_common.cuh"

namespace simnet {

namespace {

constexpr int kItem = 8;            // samples per work item
constexpr int kC = 64;              // channels of every conv layer (C3)
constexpr uint32_t kR1 = 128 * 1024;
constexpr uint32_t kR2 = 64 * 1024;
constexpr int kRing = 4;
constexpr int kThreadsCC = 320;

// byte offset of element (row r, float k) in a K-major SW128 tile of 128 rows
// whose K extent is split into 128-byte chunks of 32 floats (chunk-major).
__device__ __forceinline__ uint32_t sw128_f32(int r, int k) {
  const int chunk = k >> 5, kk = k & 31;
  return chunk * (128 * 128) + r * 128 + ((((kk >> 2) ^ (r & 7)) << 4) | ((kk & 3) << 2));
}
// same for bf16 (64 elements per chunk), offset of the 16-byte unit holding k..k+7
__device__ __forceinline__ uint32_t sw128_bf16_unit(int r, int k) {
  const int chunk = k >> 6, kk = k & 63;
  return chunk * (128 * 128) + r * 128 + (((kk >> 3) ^ (r & 7)) << 4);
}

template <int kMode>
struct ChainShape {
  static constexpr bool kSplit = kMode == kTF32x3;
  static constexpr int kElems = kMode == kBF16 ? 64 : 32;      // elements per 128 B chunk
  static constexpr int kK0Chunks = kMode == kBF16 ? 2 : 4;     // conv0 K = 100 (+pad)
  static constexpr int kK0Steps = kMode == kBF16 ? 7 : 13;     // 32 B MMA k-steps covering K = 100
  static constexpr int kKChunks = kMode == kBF16 ? 2 : 4;      // conv1/2 K = 128
  static constexpr uint32_t kWBytes = kC * 128 * kKChunks;     // one weight copy (hi or lo)
  static constexpr uint32_t kStage = 128 * 128;                // one A chunk
  static constexpr uint32_t kALo = kKChunks * kStage;          // offset of the lo copy of a restaged A
  static constexpr uint32_t kWChunk = kC * 128 * (kSplit ? 2 : 1);  // per K chunk: hi rows (+ lo rows)
  static constexpr uint32_t kAccW = kSplit ? 2 * kC : kC;
  static constexpr uint32_t kConv1Col = kSplit ? 0 : 256;
  static constexpr uint32_t kConv2Col = kSplit ? 256 : 384;
};

// Restage 64 accumulator columns of TMEM lane-row `tl` (one conv output row)
// into the A operand at row `ar`, K offset `k0`, with bias + ReLU.
template <int kMode>
__device__ __forceinline__ void restage_row(uint8_t* a, uint32_t tl, int ar, int k0, const float* bias) {
  using S = ChainShape<kMode>;
  for (int c0 = 0; c0 < kC; c0 += 16) {
    float v[16];
    tmem_ld16(tl + c0, v);
    if constexpr (S::kSplit) {  // + the cross half (Ahi.Wlo + Alo.Whi)
      float x[16];
      tmem_ld16(tl + kC + c0, x);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += x[i];
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + bias[c0 + i], 0.0f);
    if constexpr (kMode == kBF16) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint4 pk;
        uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * h + 2 * i], v[8 * h + 2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(a + sw128_bf16_unit(ar, k0 + c0 + 8 * h)) = pk;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + c0 + 4 * q;
        float4 hi;
        if constexpr (S::kSplit) {
          uint32_t u[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) u[i] = (__float_as_uint(v[4 * q + i]) + 0x1000u) & 0xffffe000u;
          hi = make_float4(__uint_as_float(u[0]), __uint_as_float(u[1]), __uint_as_float(u[2]), __uint_as_float(u[3]));
          const float4 lo = make_float4(v[4 * q] - hi.x, v[4 * q + 1] - hi.y, v[4 * q + 2] - hi.z, v[4 * q + 3] - hi.w);
          *reinterpret_cast<float4*>(a + S::kALo + sw128_f32(ar, k)) = lo;
        } else {
          hi = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        *reinterpret_cast<float4*>(a + sw128_f32(ar, k)) = hi;
      }
    }
  }
}

}  // namespace

template <int kMode>
__global__ void __launch_bounds__(kThreadsCC, 1)
conv_chain_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmXlo,
                  const __grid_constant__ CUtensorMap tmW0,
                  const __grid_constant__ CUtensorMap tmW0lo, const __grid_constant__ CUtensorMap tmW1,
                  const __grid_constant__ CUtensorMap tmW1lo, const __grid_constant__ CUtensorMap tmW2,
                  const __grid_constant__ CUtensorMap tmW2lo, ChainParams p) {
  using S = ChainShape<kMode>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* R1 = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
  uint8_t* R2 = R1 + kR1;
  uint8_t* ringA = R1;                                   // stage s: hi at s*kStage, lo at (kRing + s)*kStage
  __shared__ __align__(8) uint64_t full[kRing], split[kRing], empty[kRing];
  // One barrier per event, each completing exactly once per work item, so a
  // parity wait on (item & 1) is unambiguous (no waiter can fall two phases behind).
  __shared__ __align__(8) uint64_t bar_w[3];              // weights of layer l landed (TMA tx)
  __shared__ __align__(8) uint64_t bar_c0, bar_m1a, bar_m1b, bar_m2;  // MMAs done (tcgen05.commit)
  __shared__ __align__(8) uint64_t bar_a[3];              // A operand restaged for conv1 t0 / t1 / conv2
  __shared__ __align__(8) uint64_t bar_out;               // conv2 accumulator drained
  __shared__ uint32_t tmem_slot;
  __shared__ float sbias[3][kC];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = (p.samples + kItem - 1) / kItem;
  if (threadIdx.x < 3 * kC) {
    const int l = threadIdx.x / kC, c = threadIdx.x % kC;
    sbias[l][c] = (l == 0 ? p.b0 : (l == 1 ? p.b1 : p.b2))[c];
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&split[i], 128);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&bar_w[i], 1);
      mbar_init(&bar_a[i], 128);
    }
    mbar_init(&bar_c0, 1);
    mbar_init(&bar_m1a, 1);
    mbar_init(&bar_m1b, 1);
    mbar_init(&bar_m2, 1);
    mbar_init(&bar_out, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  // diagnostics: clock64 per event for the first work item of each CTA
  long long* tr = p.trace ? p.trace + blockIdx.x * 32 : nullptr;
  auto mark = [&](int i) {
    if (tr) tr[i] = clock64();
  };
  if (threadIdx.x == 0) mark(0);

  auto load_w = [&](int layer, const CUtensorMap* hi, const CUtensorMap* lo, int chunks) {
    uint64_t* b = &bar_w[layer];
    mbar_expect_tx(b, S::kWBytes * (S::kSplit ? 2u : 1u) / S::kKChunks * chunks);
    for (int c = 0; c < chunks; ++c) {
      tma_load_2d(R2 + c * S::kWChunk, hi, b, c * S::kElems, 0);
      if (S::kSplit) tma_load_2d(R2 + c * S::kWChunk + kC * 128, lo, b, c * S::kElems, 0);
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        if (it > 0) mbar_wait(&bar_m2, (it - 1) & 1);  // previous conv2 done: R1, R2 free
        load_w(0, &tmW0, &tmW0lo, S::kK0Chunks);
        if (it == 0) mark(1);
        for (int c = 0; c < 4 * S::kK0Chunks; ++c) {
          const int tile = c / S::kK0Chunks, kc = c % S::kK0Chunks;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], S::kStage * (S::kSplit ? 2u : 1u));
          tma_load_3d(ringA + stage * S::kStage, &tmX, &full[stage], kc * S::kElems, 0, item * kItem + 2 * tile);
          if (S::kSplit)  // K1 wrote the 3xTF32 lo plane next to the hi plane
            tma_load_3d(ringA + (kRing + stage) * S::kStage, &tmXlo, &full[stage], kc * S::kElems, 0,
                        item * kItem + 2 * tile);
          if (++stage == kRing) {
            stage = 0;
            phase ^= 1;
          }
        }
        mbar_wait(&bar_c0, it & 1);  // conv0 MMAs done: W0 no longer read
        if (it == 0) mark(2);
        load_w(1, &tmW1, &tmW1lo, S::kKChunks);
        mbar_wait(&bar_m1b, it & 1);  // conv1 done: W1 no longer read
        if (it == 0) mark(3);
        load_w(2, &tmW2, &tmW2lo, S::kKChunks);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = instr_desc(mode_fmt(kMode), kC);
      const uint32_t idesc2 = instr_desc(mode_fmt(kMode), 2 * kC);  // 3xTF32: Ahi x [Whi; Wlo]
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint32_t r1 = su32(R1), r2 = su32(R2);
      auto gemm_resident_a = [&](uint32_t d, int ksteps) {  // A restaged in R1, W in R2
        for (int s = 0; s < ksteps; ++s) {
          const int c = s >> 2, j = s & 3;
          const uint32_t ao = c * S::kStage + j * 32, wo = c * S::kWChunk + j * 32;
          const uint64_t ad = smem_desc_sw128(r1 + ao), bd = smem_desc_sw128(r2 + wo);
          if (S::kSplit) {
            mma<kMode>(d, ad, bd, idesc2, s > 0);
            mma<kMode>(d + kC, smem_desc_sw128(r1 + S::kALo + ao), bd, idesc, 1);
          } else {
            mma<kMode>(d, ad, bd, idesc, s > 0);
          }
        }
      };
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        // conv0: 4 tiles of 128 rows (2 samples each) streamed through the ring
        mbar_wait(&bar_w[0], it & 1);
        if (it == 0) mark(4);
        if (S::kSplit && it > 0) mbar_wait(&bar_out, (it - 1) & 1);  // conv0 tile 2 overwrites the conv2 columns
        tc_fence_after();
        for (int tile = 0; tile < 4; ++tile) {
          const uint32_t d = tmem + tile * S::kAccW;
          for (int kc = 0; kc < S::kK0Chunks; ++kc) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const int steps = kc == S::kK0Chunks - 1 ? S::kK0Steps - 4 * (S::kK0Chunks - 1) : 4;
            for (int j = 0; j < steps; ++j) {
              const uint32_t ao = su32(ringA) + stage * S::kStage + j * 32;
              const uint32_t wo = r2 + kc * S::kWChunk + j * 32;
              const uint32_t acc = (kc == 0 && j == 0) ? 0u : 1u;
              if (S::kSplit) {
                mma<kMode>(d, smem_desc_sw128(ao), smem_desc_sw128(wo), idesc2, acc);
                mma<kMode>(d + kC, smem_desc_sw128(ao + kRing * S::kStage), smem_desc_sw128(wo), idesc, 1);
              } else {
                mma<kMode>(d, smem_desc_sw128(ao), smem_desc_sw128(wo), idesc, acc);
              }
            }
            mma_commit(&empty[stage]);
            if (++stage == kRing) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        mma_commit(&bar_c0);
        if (it == 0) mark(5);
        // conv1: two tiles of 128 rows (4 samples each), A restaged by the epilogue
        mbar_wait(&bar_a[0], it & 1);
        if (it == 0) mark(6);
        mbar_wait(&bar_w[1], it & 1);
        if (it == 0) mark(7);
        tc_fence_after();
        gemm_resident_a(tmem + S::kConv1Col, 4 * S::kKChunks);
        mma_commit(&bar_m1a);
        mbar_wait(&bar_a[1], it & 1);
        if (it == 0) mark(8);
        tc_fence_after();
        gemm_resident_a(tmem + S::kConv1Col + S::kAccW, 4 * S::kKChunks);
        mma_commit(&bar_m1b);
        // conv2: one tile of 128 rows (8 samples)
        mbar_wait(&bar_a[2], it & 1);
        if (it == 0) mark(9);
        mbar_wait(&bar_w[2], it & 1);
        if (it == 0) mark(10);
        if (it > 0) mbar_wait(&bar_out, (it - 1) & 1);  // previous conv2 accumulator drained
        tc_fence_after();
        gemm_resident_a(tmem + S::kConv2Col, 4 * S::kKChunks);
        mma_commit(&bar_m2);
        if (it == 0) mark(11);
      }
    }
    __syncwarp();
  } else if (warp < 6) {
    // warps 2-5: spare (the 3xTF32 split of the input now happens in K1)
  } else {
    // epilogue warps 6..9: thread owns TMEM lane m = 32*(warp%4) + lane
    const int quad = warp & 3;
    const int m = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      // A1 passes: conv0 tiles (2*pass, 2*pass+1) -> conv1 A rows
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 0)
          mbar_wait(&bar_c0, it & 1);
        else
          mbar_wait(&bar_m1a, it & 1);  // conv1 tile 0 has consumed R1
        tc_fence_after();
        for (int t2 = 0; t2 < 2; ++t2) {
          // conv0 row m of tile (2*pass + t2) = (sample, pos) -> A1 row t2*64 + m/2, K half m%2
          restage_row<kMode>(R1, tmem + lane_off + (2 * pass + t2) * S::kAccW, t2 * 64 + (m >> 1), (m & 1) * kC,
                             sbias[0]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&bar_a[pass]);
      }
      // A2: conv1 tiles 0,1 -> conv2 A rows
      mbar_wait(&bar_m1b, it & 1);
      tc_fence_after();
      for (int t2 = 0; t2 < 2; ++t2)
        restage_row<kMode>(R1, tmem + lane_off + S::kConv1Col + t2 * S::kAccW, t2 * 64 + (m >> 1), (m & 1) * kC,
                           sbias[1]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&bar_a[2]);
      // conv2 -> flat[sample][pos*64 + c]: row m of the tile is flat row item*128 + m
      mbar_wait(&bar_m2, it & 1);
      if (it == 0 && m == 0) mark(12);
      tc_fence_after();
      const int sample = item * kItem + (m >> 4);
      for (int c0 = 0; c0 < kC; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + lane_off + S::kConv2Col + c0, v);
        if constexpr (S::kSplit) {
          float x[16];
          tmem_ld16(tmem + lane_off + S::kConv2Col + kC + c0, x);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += x[i];
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + sbias[2][c0 + i], 0.0f);
        if (sample < p.samples) {
          const uint64_t off = static_cast<uint64_t>(item) * (kItem * 16 * kC) + m * kC + c0;
          if (kMode == kBF16) {
            uint4 pk[2];
            uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
              w[i] = *reinterpret_cast<uint32_t*>(&b2);
            }
            uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + off);
            o[0] = pk[0];
            o[1] = pk[1];
          } else {
            float4* o = reinterpret_cast<float4*>(static_cast<float*>(p.out) + off);
#pragma unroll
            for (int i = 0; i < 4; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bar_out);
      if (it == 0 && m == 0) mark(13);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

size_t chain_smem_bytes() { return kR1 + kR2 + 1024; }

void launch_conv_chain(int mode, const CUtensorMap& x, const CUtensorMap& xlo, const CUtensorMap* w,
                       const ChainParams& p, int num_sms, cudaStream_t s) {
  const int items = (p.samples + kItem - 1) / kItem;
  const dim3 grid(static_cast<unsigned>(items < num_sms ? items : num_sms));
  const size_t sm = chain_smem_bytes();
  if (mode == kBF16)
    conv_chain_kernel<kBF16><<<grid, kThreadsCC, sm, s>>>(x, xlo, w[0], w[1], w[2], w[3], w[4], w[5], p);
  else if (mode == kTF32)
    conv_chain_kernel<kTF32><<<grid, kThreadsCC, sm, s>>>(x, xlo, w[0], w[1], w[2], w[3], w[4], w[5], p);
  else
    conv_chain_kernel<kTF32x3><<<grid, kThreadsCC, sm, s>>>(x, xlo, w[0], w[1], w[2], w[3], w[4], w[5], p);
}

void conv_chain_set_attributes() {
  const int sm = static_cast<int>(chain_smem_bytes());
  CUDA_OK(cudaFuncSetAttribute(conv_chain_kernel<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(conv_chain_kernel<kTF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(conv_chain_kernel<kTF32x3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
}

}  // namespace simnet
