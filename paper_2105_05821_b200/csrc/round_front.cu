// Fused round front = K1 + the conv chain of K2, one kernel per round.
//
// Per work item (8 sub-traces), in one CTA:
//   1. apply   — warp w applies the pending step of sub-trace w (retire /
//                stall / push / drain, simcore.cpp:112-159) and builds its
//                context-column table (next_request, simcore.cpp:25-66):
//                instruction index + the 9 dynamic slots, newest first.
//   2. gather  — the 256 compute threads write the normalised input straight
//                into the conv0 A operand (K-major SWIZZLE_128B, 3xTF32 hi/lo
//                planes or bf16) in shared memory.  conv0 tiles are
//                row-major over (sample, row-of-two-columns): tile t holds rows
//                16t..16t+15 of all 8 samples, so a tile beyond every
//                sample's context is all zeros and is skipped: its conv0
//                output is exactly ReLU(b0) (a zero row accumulates exactly 0).
//   3. conv0 -> conv1 -> conv2 on tcgen05 with TMEM accumulators and the
//                epilogue restaging each layer's output as the next A operand
//                (cnn.cpp:90-110), as in conv_chain.cu.  Only the final conv2
//                activations (4 KB / sample) leave the SM.
// Per-row results are identical to the unfused path (ctx_kernel + TMA
// conv_chain_kernel): every accumulator row depends only on its own A row.
//
//   TMEM (f32 columns): conv0 4 x 64 [0,256) | conv1 2 x 64 [256,384) | conv2 [384,448);
//   3xTF32: every tile's accumulator is 128 columns, [Ahi.Whi | Ahi.Wlo + Alo.Whi]
//   (one N = 128 MMA of Ahi against the stacked [Whi; Wlo] plus one N = 64
//   MMA of Alo, summed by the epilogue): conv0 t at 128t, conv1 u at 128u
//   (over conv0 tiles already restaged), conv2 at 256.
//   SMEM: R1 128 KB  conv0 A tile (hi | lo) / restaged conv1 / conv2 A tile
//         R2  64 KB  current layer's weights (hi | lo), TMA
//         T   20 KB  column tables
//   warps 0-7   compute: apply, gather, epilogue (TMEM lane quarter w%4)
//   warp 8      TMA producer (weights)
//   warp 9      TMEM allocator + tcgen05.mma issuer
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>

#include <cstdlib>

#include "conv_chain.cuh"
#include "k1_device.cuh"
#include "launch.cuh"
#include "round_front.cuh"
#include "tc_common.cuh"

namespace simnet {

namespace {

constexpr int kItem = 8;      // sub-traces per work item
constexpr int kC = 64;        // channels of every conv layer (C3)
constexpr int kRowsT = 16;    // conv0 rows per sample per tile
constexpr int kTblCols = 128; // max columns (max_context + 1)
constexpr uint32_t kR1 = 128 * 1024;
constexpr uint32_t kR2 = 64 * 1024;
constexpr uint32_t kTbl = kItem * kTblCols * (4 + 16);
constexpr uint32_t kOutStage = 96 * 1024;  // flat staging in R1 (2 x 16 KB)
// Tile-0 static-slot staging in R1 during the decode (R1 holds W2 [0, 64 KB)
// and h / y [64 KB, 74 KB) then): per sample one TMA box of 32 trace rows
// [lo, lo + 32) ending at the predicted target, 176 B per row (11 x 16 B: an
// odd pitch, so LDS.128 of 8 rows hit 8 distinct bank groups).  It starts past
// conv0's K chunk 0 (hi [0, 16 KB), lo [64, 80 KB)), so tile 0's chunk-0
// stores need not wait for the other threads' staging reads.
constexpr uint32_t kStgOff = 80 * 1024;
static_assert(kStgOff + kItem * 32 * 176 <= kR1, "tile-0 staging must fit in R1");
constexpr uint32_t kStgPitch = 176;
constexpr uint32_t kStgBox = 32 * kStgPitch;  // 5632 B, 128-B aligned
constexpr int kThreadsRF = 320;
constexpr int kCompute = 256;

__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }


// byte offset of f32 element (row r, k) in a K-major SW128 tile of 128 rows
// whose K extent is split into chunk-major 128-byte chunks of 32 floats.
__device__ __forceinline__ uint32_t sw128_f32(int r, int k) {
  const int chunk = k >> 5, kk = k & 31;
  return chunk * (128 * 128) + r * 128 + ((((kk >> 2) ^ (r & 7)) << 4) | ((kk & 3) << 2));
}
// bf16 element (row r, k), 64 elements per chunk
__device__ __forceinline__ uint32_t sw128_bf16(int r, int k) {
  const int chunk = k >> 6, kk = k & 63;
  return chunk * (128 * 128) + r * 128 + ((((kk >> 3) ^ (r & 7)) << 4) | ((kk & 7) << 1));
}

// fp8 e4m3 element (row r, k), 128 elements per chunk
__device__ __forceinline__ uint32_t sw128_fp8(int r, int k) {
  const int chunk = k >> 7, kk = k & 127;
  return chunk * (128 * 128) + r * 128 + ((((kk >> 4) ^ (r & 7)) << 4) | (kk & 15));
}
__device__ __forceinline__ uint16_t fp8x2(float v0, float v1) {
  return static_cast<uint16_t>(__nv_cvt_float2_to_fp8x2(make_float2(v0, v1), __NV_SATFINITE, __NV_E4M3));
}

template <int kMode>
struct Shape {
  static constexpr bool kSplit = kMode == kTF32x3;
  static constexpr int kElems = mode_chunk_elems(kMode);                           // elements per 128 B chunk
  static constexpr int kK0Chunks = kMode == kFP8 ? 1 : (kMode == kBF16 ? 2 : 4);   // conv0 K = 100 (+pad)
  static constexpr int kK0Steps = kMode == kFP8 ? 4 : (kMode == kBF16 ? 7 : 13);   // 32 B k-steps covering K = 100
  static constexpr int kPadUnits = kMode == kFP8 ? 14 : (kMode == kBF16 ? 6 : 2);  // pairs of zeros after K = 100
  static constexpr int kKChunks = kMode == kFP8 ? 1 : (kMode == kBF16 ? 2 : 4);    // conv1/2 K = 128
  static constexpr uint32_t kWBytes = kC * 128 * kKChunks;  // one weight copy (hi or lo)
  // 3xTF32 weights: per K chunk the 64 hi rows then the 64 lo rows (16 KB), so
  // [Whi; Wlo] is one N = 128 B operand; other modes: one 8 KB chunk per K chunk
  static constexpr uint32_t kWChunk = kC * 128 * (kSplit ? 2 : 1);
  static constexpr uint32_t kAccW = kSplit ? 2 * kC : kC;     // TMEM columns per tile accumulator
  static constexpr uint32_t kConv1Col = kSplit ? 0 : 256;     // conv1 tile u at kConv1Col + u * kAccW
  static constexpr uint32_t kConv2Col = kSplit ? 256 : 384;
  static constexpr uint32_t kStage = 128 * 128;             // one A chunk (128 rows x 128 B)
  static constexpr uint32_t kALo = kKChunks * kStage;       // lo plane of a restaged A
  static constexpr uint32_t kA0Lo = 4 * kStage;             // lo plane of the conv0 A tile
};

// Store the float pair (v0, v1) of A row r at K offset k (even) into the
// operand planes: 3xTF32 hi = cvt.rna, lo = v - hi (exact); tf32 plain; bf16 rn.
template <int kMode>
__device__ __forceinline__ void put2(uint8_t* a, uint32_t lo_off, int r, int k, float v0, float v1) {
  if constexpr (kMode == kFP8) {
    *reinterpret_cast<uint16_t*>(a + sw128_fp8(r, k)) = fp8x2(v0, v1);
  } else if constexpr (kMode == kBF16) {
    __nv_bfloat162 b = __floats2bfloat162_rn(v0, v1);
    *reinterpret_cast<__nv_bfloat162*>(a + sw128_bf16(r, k)) = b;
  } else {
    const uint32_t o = sw128_f32(r, k);
    if constexpr (kMode == kTF32x3) {
      const float h0 = __uint_as_float((__float_as_uint(v0) + 0x1000u) & 0xffffe000u);
      const float h1 = __uint_as_float((__float_as_uint(v1) + 0x1000u) & 0xffffe000u);
      *reinterpret_cast<float2*>(a + o) = make_float2(h0, h1);
      *reinterpret_cast<float2*>(a + lo_off + o) = make_float2(v0 - h0, v1 - h1);
    } else {
      *reinterpret_cast<float2*>(a + o) = make_float2(v0, v1);
    }
  }
}

// Four floats of A row r at K offset k (multiple of 4): one 16-B store per plane.
template <int kMode>
__device__ __forceinline__ void put4(uint8_t* a, uint32_t lo_off, int r, int k, float v0, float v1, float v2,
                                     float v3) {
  if constexpr (kMode == kFP8) {
    *reinterpret_cast<uint32_t*>(a + sw128_fp8(r, k)) =
        static_cast<uint32_t>(fp8x2(v0, v1)) | (static_cast<uint32_t>(fp8x2(v2, v3)) << 16);
  } else if constexpr (kMode == kBF16) {
    put2<kMode>(a, lo_off, r, k, v0, v1);
    put2<kMode>(a, lo_off, r, k + 2, v2, v3);
  } else {
    const uint32_t o = sw128_f32(r, k);
    if constexpr (kMode == kTF32x3) {
      float4 hi;
      hi.x = __uint_as_float((__float_as_uint(v0) + 0x1000u) & 0xffffe000u);
      hi.y = __uint_as_float((__float_as_uint(v1) + 0x1000u) & 0xffffe000u);
      hi.z = __uint_as_float((__float_as_uint(v2) + 0x1000u) & 0xffffe000u);
      hi.w = __uint_as_float((__float_as_uint(v3) + 0x1000u) & 0xffffe000u);
      *reinterpret_cast<float4*>(a + o) = hi;
      *reinterpret_cast<float4*>(a + lo_off + o) = make_float4(v0 - hi.x, v1 - hi.y, v2 - hi.z, v3 - hi.w);
    } else {
      *reinterpret_cast<float4*>(a + o) = make_float4(v0, v1, v2, v3);
    }
  }
}

// Restage 64 accumulator columns of TMEM lane-row `tl` (one conv output row)
// into the A operand at row `ar`, K offset `k0`, with bias + ReLU.  `accv`
// non-null: the accumulator row is given (a skipped all-zero conv0 row is
// exactly 0; a skipped all-constant conv1 row is the calibrated c1acc).
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// Row order inside each sample's 16 rows of a tile.  Each restage lane pair
// (positions 2j, 2j+1) lands in ONE next-layer row (K halves 0 and 64 share
// banks), so a layer's rows are ordered so that every quarter-warp of the
// restage (8 consecutive TMEM lanes) writes 8 distinct rows with distinct
// swizzle phases: conflict-free 16-B stores.
//   conv0: slot s holds position 2(s%8) + s/8 (evens in 0-7, odds in 8-15);
//   conv1: position p sits in slot conv1_slot(p) (evens p/2, odds 8 + (p/2 ^ 4));
//   conv2: natural (slot = position), so flat needs no reordering.
__device__ __forceinline__ int conv1_slot(int p) { return (p & 1) ? 8 + ((p >> 1) ^ 4) : (p >> 1); }

// 16 accumulator values (raw f32 bits, columns c0..c0+15 of the row) ->
// bias + ReLU -> the next layer's A operand at row `ar`, K offset k0 + c0.
template <int kMode>
__device__ __forceinline__ void restage16(uint8_t* a, const uint32_t* raw, int c0, int ar, int k0,
                                          const float* bias, float scale) {
  using S = Shape<kMode>;
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float x = __uint_as_float(raw[i]);
    if constexpr (kMode == kFP8) x *= scale;  // undo the weight scale
    v[i] = fmaxf(x + bias[c0 + i], 0.0f);
  }
  if constexpr (kMode == kFP8) {  // 16 e4m3 values: one 16-B unit of row ar
    uint4 pk;
    uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      w[i] = static_cast<uint32_t>(fp8x2(v[4 * i], v[4 * i + 1])) |
             (static_cast<uint32_t>(fp8x2(v[4 * i + 2], v[4 * i + 3])) << 16);
    *reinterpret_cast<uint4*>(a + ar * 128 + ((((k0 + c0) >> 4) ^ (ar & 7)) << 4)) = pk;
  } else if constexpr (kMode == kBF16) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint4 pk;
      uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * h + 2 * i], v[8 * h + 2 * i + 1]);
        w[i] = *reinterpret_cast<uint32_t*>(&b2);
      }
      const int k = k0 + c0 + 8 * h;
      const int chunk = k >> 6, kk = k & 63;
      *reinterpret_cast<uint4*>(a + chunk * (128 * 128) + ar * 128 + (((kk >> 3) ^ (ar & 7)) << 4)) = pk;
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

template <int kMode>
__device__ __forceinline__ void restage_row(uint8_t* a, uint32_t tl, const float* accv, int ar, int k0,
                                            const float* bias, float scale) {
  using S = Shape<kMode>;
  if constexpr (S::kSplit) {
    // [hi.hi | cross] accumulator: per 32 columns both halves in flight, one
    // wait, summed (hi.hi + cross), restaged; not unrolled (instruction-fetch
    // stalls dominate this phase: one body is half the code)
#pragma unroll 1
    for (int h = 0; h < kC; h += 32) {
      uint32_t raw[32];
      if (accv) {  // accumulator row known in advance (shared memory), no TMEM read
#pragma unroll
        for (int i = 0; i < 32; ++i) raw[i] = __float_as_uint(accv[h + i]);
      } else {
        uint32_t x[32];
        tmem_ld16_async(tl + h, raw);
        tmem_ld16_async(tl + h + 16, raw + 16);
        tmem_ld16_async(tl + kC + h, x);
        tmem_ld16_async(tl + kC + h + 16, x + 16);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; ++i) raw[i] = __float_as_uint(__uint_as_float(raw[i]) + __uint_as_float(x[i]));
      }
      restage16<kMode>(a, raw, h, ar, k0, bias, scale);
      restage16<kMode>(a, raw + 16, h + 16, ar, k0, bias, scale);
    }
    return;
  }
  uint32_t raw[kC];
  if (accv) {  // accumulator row known in advance (shared memory), no TMEM read
#pragma unroll
    for (int i = 0; i < kC; ++i) raw[i] = __float_as_uint(accv[i]);
  } else {  // all four 16-column loads in flight, one wait
#pragma unroll
    for (int c0 = 0; c0 < kC; c0 += 16) tmem_ld16_async(tl + c0, raw + c0);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
#pragma unroll
  for (int c0 = 0; c0 < kC; c0 += 16) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float x = __uint_as_float(raw[c0 + i]);
      if constexpr (kMode == kFP8) x *= scale;  // undo the weight scale
      v[i] = fmaxf(x + bias[c0 + i], 0.0f);
    }
    if constexpr (kMode == kFP8) {  // 16 e4m3 values: one 16-B unit of row ar
      uint4 pk;
      uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        w[i] = static_cast<uint32_t>(fp8x2(v[4 * i], v[4 * i + 1])) |
               (static_cast<uint32_t>(fp8x2(v[4 * i + 2], v[4 * i + 3])) << 16);
      *reinterpret_cast<uint4*>(a + ar * 128 + ((((k0 + c0) >> 4) ^ (ar & 7)) << 4)) = pk;
    } else if constexpr (kMode == kBF16) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint4 pk;
        uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * h + 2 * i], v[8 * h + 2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
        const int k = k0 + c0 + 8 * h;
        const int chunk = k >> 6, kk = k & 63;
        *reinterpret_cast<uint4*>(a + chunk * (128 * 128) + ar * 128 + (((kk >> 3) ^ (ar & 7)) << 4)) = pk;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + c0 + 4 * q;
        const float4 hi = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        *reinterpret_cast<float4*>(a + sw128_f32(ar, k)) = hi;
      }
    }
  }
}

}  // namespace

// kMulti: the launch gives CTAs several items (K > 8 x SMs); later items get
// their FC1 partial rows bulk-copied into R2 during the previous item's tail.
// A separate instantiation, so the single-item kernel's code is untouched.
template <int kMode, bool kMulti>
__global__ void __launch_bounds__(kThreadsRF, 1)
round_front_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW0lo,
                   const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW1lo,
                   const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmW2lo,
                   const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmStat,
                   FrontParams p) {
  using S = Shape<kMode>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* R1 = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
  uint8_t* R2 = R1 + kR1;
  uint32_t* tbl_inst = reinterpret_cast<uint32_t*>(R2 + kR2);                // [kItem][kTblCols]
  float4* tbl_dyn = reinterpret_cast<float4*>(tbl_inst + kItem * kTblCols);  // [kItem][kTblCols]
  // One barrier per event kind; each waiter consumes every completion in order.
  __shared__ __align__(8) uint64_t bar_w[3];       // layer weights landed (TMA tx), 1 / item
  __shared__ __align__(8) uint64_t bar_a0, bar_t0; // conv0 tile gathered (256) / its MMAs done: T / item
  // f32 modes: conv0 tile K chunk c (32 floats) written; the MMAs of a chunk
  // start while later chunks are still being stored.  Writers: chunk 0 the
  // even-column threads (K 0-49), 1 both, 2-3 the odd-column threads (K 50-103)
  __shared__ __align__(8) uint64_t bar_a0c[4];
  __shared__ __align__(8) uint64_t bar_c0;         // all conv0 MMAs done (W0 + conv0 A free), 1 / item
  __shared__ __align__(8) uint64_t bar_a1, bar_m1; // conv1 A restaged / its MMAs done: 2 / item
  __shared__ __align__(8) uint64_t bar_w1f;        // conv1 MMAs done (W1 free), 1 / item
  __shared__ __align__(8) uint64_t bar_a2, bar_m2; // conv2 A restaged / MMAs done: 1 / item
  __shared__ __align__(8) uint64_t bar_w2;         // FC2 weights landed in R1 (bulk copy), 1 / item
  __shared__ __align__(8) uint64_t bar_st;         // the item's SubStates landed (bulk copy), 1 / item
  __shared__ __align__(16) SubState s_state[kItem];
  __shared__ __align__(8) uint64_t bar_tg;         // the items' next-target pc / address / flags prefetched
  __shared__ uint64_t s_tidx[kItem], s_tpc[kItem], s_taddr[kItem];
  __shared__ uint32_t s_tfl[kItem];
  __shared__ __align__(8) uint64_t bar_stg;        // tile-0 static rows staged in R1 (bulk copies)
  __shared__ __align__(8) uint64_t bar_fo;         // flat-output staging in R1 read back (8 warps), 1 / item
  __shared__ __align__(8) uint64_t bar_part;       // the item's FC1 split-K partial rows landed in R2, 1 / item
  __shared__ __align__(8) uint64_t bar_pread;      // ... and were read by the decode (256): R2 free for W0
  __shared__ uint32_t s_stg_lo[kItem], s_stg_hi[kItem];  // staged trace-row range per sample (hi - row = slot)
  __shared__ uint32_t tmem_slot;
  __shared__ float sbias[3][kC];
  __shared__ float s_zero[kSlots], s_one[kSlots];
  __shared__ int s_ncols[kItem];  // context columns of each sample this round, -1: inactive
  __shared__ int s_T;             // conv0 tiles needed this item
  __shared__ float s_zacc[kC];    // zero accumulator row (skipped conv0 tiles)
  __shared__ float s_c1[kC];      // calibrated conv1 accumulator of a constant row
  __shared__ double s_lab[6];     // label mean / stdev (decode)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t samples = p.last - p.first;
  const int n_items = static_cast<int>((samples + kItem - 1) / kItem);
  // PDL: the FC kernels may launch now (their prologue only touches weights);
  // this kernel's prologue (barriers, TMEM, biases, W0) overlaps the previous
  // round's tail, and only the compute warps wait for its results.
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 32 + 30] = global_ns();  // diagnostics: CTA entry
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x < 3 * kC) {
    const int l = threadIdx.x / kC, c = threadIdx.x % kC;
    sbias[l][c] = (l == 0 ? p.b0 : (l == 1 ? p.b1 : p.b2))[c];
  } else if (threadIdx.x < 3 * kC + kSlots) {
    const int k = threadIdx.x - 3 * kC;
    s_zero[k] = p.nc ? p.nc->zero[k] : 0.0f;
    s_one[k] = p.nc ? p.nc->one[k] : 0.0f;
  } else if (threadIdx.x >= 256 && threadIdx.x < 256 + kC) {
    const int k = threadIdx.x - 256;
    s_zacc[k] = 0.0f;
    s_c1[k] = p.c1acc ? p.c1acc[k] : 0.0f;
  } else if (threadIdx.x >= 3 * kC + kSlots && threadIdx.x < 3 * kC + kSlots + 6) {
    const int k = threadIdx.x - 3 * kC - kSlots;
    s_lab[k] = p.nc ? (k < 3 ? p.nc->label_mean[k] : p.nc->label_sd[k - 3]) : 0.0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar_w[i], 1);
    mbar_init(&bar_a0, kCompute);
    mbar_init(&bar_a0c[0], kCompute / 2);
    mbar_init(&bar_a0c[1], kCompute);
    mbar_init(&bar_a0c[2], kCompute / 2);
    mbar_init(&bar_a0c[3], kCompute / 2);
    mbar_init(&bar_t0, 1);
    mbar_init(&bar_c0, 1);
    mbar_init(&bar_a1, kCompute);
    mbar_init(&bar_m1, 1);
    mbar_init(&bar_w1f, 1);
    mbar_init(&bar_a2, kCompute);
    mbar_init(&bar_m2, 1);
    mbar_init(&bar_w2, 1);
    mbar_init(&bar_st, 1);
    mbar_init(&bar_tg, 1);
    mbar_init(&bar_stg, 1);
    mbar_init(&bar_fo, kCompute / 32);
    mbar_init(&bar_part, 1);
    mbar_init(&bar_pread, kCompute);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    if (p.trace && lane == 0) p.trace[blockIdx.x * 32 + 29] = global_ns();  // diagnostics: TMEM allocated
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 32 + 13] = global_ns();  // diagnostics: kernel span

  if (warp == 8) {
    // ---------------- TMA producer: layer weights ----------------
    if (lane == 0) {
      auto load_w = [&](int layer, const CUtensorMap* hi, const CUtensorMap* lo, int chunks) {
        uint64_t* b = &bar_w[layer];
        mbar_expect_tx(b, S::kWBytes * (S::kSplit ? 2u : 1u) / S::kKChunks * chunks);
        for (int c = 0; c < chunks; ++c) {
          tma_load_2d(R2 + c * S::kWChunk, hi, b, c * S::kElems, 0);
          if (S::kSplit) tma_load_2d(R2 + c * S::kWChunk + kC * 128, lo, b, c * S::kElems, 0);
        }
      };
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        if (it > 0) mbar_wait(&bar_m2, (it - 1) & 1);  // previous conv2 done: R1, R2 free
        {  // FC2 weights for the decode of the previous round's predictions (R1 is idle until the gather)
          const uint32_t bytes = static_cast<uint32_t>(p.fc.od * p.fc.hidden * 4);
          if (bytes == 0) {
            mbar_arrive(&bar_w2);
          } else {
            mbar_expect_tx(&bar_w2, bytes);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(R1)),
                "l"(p.fc.w2t), "r"(bytes), "r"(su32(&bar_w2))
                : "memory");
          }
        }
        if (it == 0) load_w(0, &tmW0, &tmW0lo, S::kK0Chunks);  // a constant: ahead of the dependency wait
        {  // the item's sub-trace states, contiguous in HBM: one bulk copy, ahead of the decode
          if (it == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // previous round final (PDL)
          const uint64_t s0 = p.first + static_cast<uint64_t>(item) * kItem;
          const uint64_t cnt = p.calibrate ? 0 : (p.last - s0 < kItem ? p.last - s0 : kItem);
          if (kMulti && it > 0) {
            // later items: the item's rows of the FC1 split-K partial planes -> R2
            // [q][8][hidden] right after the previous item's conv2 (W0 comes after
            // the decode has read them).  The first item reads them with direct
            // loads: at kernel start the TMA unit is busy with W2, W0 and the staging.
            const uint32_t row_bytes = static_cast<uint32_t>(p.fc.hidden) * 4u;
            const uint32_t bytes = static_cast<uint32_t>(cnt) * row_bytes;
            mbar_expect_tx(&bar_part, bytes * static_cast<uint32_t>(p.fc.nsplit));
            for (int q = 0; q < p.fc.nsplit && bytes > 0; ++q)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      su32(R2 + q * kItem * row_bytes)),
                  "l"(p.fc.part + q * p.fc.split_stride + (s0 - p.first) * p.fc.hidden), "r"(bytes),
                  "r"(su32(&bar_part))
                  : "memory");
          }
          const uint32_t bytes = static_cast<uint32_t>(cnt * sizeof(SubState));
          if (bytes == 0) {
            mbar_arrive(&bar_st);
          } else {
            mbar_expect_tx(&bar_st, bytes);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(s_state)),
                "l"(p.state + s0), "r"(bytes), "r"(su32(&bar_st))
                : "memory");
          }
          // Each sub-trace's next gather target is pos (+1 when this round
          // first applies a step): prefetch its pc / address / flags for the
          // column table while the compute warps run the decode.
          mbar_wait(&bar_st, it & 1);
          uint64_t idx[kItem], tpc[kItem], tad[kItem];
          uint32_t tfl[kItem];
          {  // stage the tile-0 static rows: trace rows [max(begin, target - 31), target]
            if (it > 0) mbar_wait(&bar_fo, (it - 1) & 1);  // previous item's flat staging (R1 96 KB+) read
            uint32_t total = 0;
#pragma unroll
            for (int w = 0; w < kItem; ++w) {
              const SubState& ss = s_state[w];
              const uint32_t pos = ss.pos + ((ss.awaiting || ss.has_pend) ? 1u : 0u);
              const bool ok = w < static_cast<int>(cnt) && ss.status == kOk && pos < ss.len;
              const uint32_t hi = ok ? static_cast<uint32_t>(ss.begin + pos) : 0u;
              const uint32_t lo = ok ? (pos >= 31u ? hi - 31u : static_cast<uint32_t>(ss.begin)) : 1u;
              s_stg_lo[w] = lo;
              s_stg_hi[w] = ok ? lo + 31u : 0u;  // the whole box (rows past the trace read as zeros)
              total += ok ? kStgBox : 0u;
            }
            mbar_expect_tx(&bar_stg, total);  // arrives: the ranges above are released with it
#pragma unroll 1
            for (int w = 0; w < kItem; ++w)
              if (s_stg_lo[w] <= s_stg_hi[w])
                tma_load_2d(R1 + kStgOff + w * kStgBox, &tmStat, &bar_stg, 0, static_cast<int>(s_stg_lo[w]));
          }
#pragma unroll
          for (int w = 0; w < kItem; ++w) {
            const SubState& ss = s_state[w];
            const uint32_t pos = ss.pos + ((ss.awaiting || ss.has_pend) ? 1u : 0u);
            const bool ok = w < static_cast<int>(cnt) && ss.status == kOk && pos < ss.len;
            idx[w] = ok ? ss.begin + pos : ~0ull;
            const uint64_t at = ok ? idx[w] : 0ull;
            tpc[w] = ok ? p.pc[at] : 0ull;
            tad[w] = ok ? p.addr[at] : 0ull;
            tfl[w] = ok ? p.iflags[at] : 0u;
          }
#pragma unroll
          for (int w = 0; w < kItem; ++w) {
            s_tidx[w] = idx[w];
            s_tpc[w] = tpc[w];
            s_taddr[w] = tad[w];
            s_tfl[w] = tfl[w];
          }
          mbar_arrive(&bar_tg);  // release: the smem stores above are visible to waiters
        }
        if (kMulti && it > 0) {
          mbar_wait(&bar_pread, (it - 1) & 1);  // the decode has read the partials: R2 takes W0
          load_w(0, &tmW0, &tmW0lo, S::kK0Chunks);
        }
        mbar_wait(&bar_c0, it & 1);  // conv0 MMAs done: W0 no longer read
        load_w(1, &tmW1, &tmW1lo, S::kKChunks);
        mbar_wait(&bar_w1f, it & 1);  // conv1 MMAs done: W1 no longer read
        load_w(2, &tmW2, &tmW2lo, S::kKChunks);
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = instr_desc(mode_fmt(kMode), kC);
      const uint32_t idesc2 = instr_desc(mode_fmt(kMode), 2 * kC);  // 3xTF32: Ahi x [Whi; Wlo]
      const uint32_t r1 = su32(R1), r2 = su32(R2);
      uint32_t n_a0 = 0, n_a1 = 0;
      int it = 0;
      auto gemm = [&](uint32_t d, uint32_t alo, int ksteps) {  // A in R1 (lo plane at +alo), W in R2
        for (int s = 0; s < ksteps; ++s) {
          const int c = s >> 2, j = s & 3;
          const uint32_t ao = c * S::kStage + j * 32, wo = c * S::kWChunk + j * 32;
          const uint64_t ad = smem_desc_sw128(r1 + ao), bd = smem_desc_sw128(r2 + wo);
          if (S::kSplit) {
            mma<kMode>(d, ad, bd, idesc2, s > 0);                            // [hi.hi | hi.lo]
            mma<kMode>(d + kC, smem_desc_sw128(r1 + alo + ao), bd, idesc, 1);  // cross half += lo.hi
          } else {
            mma<kMode>(d, ad, bd, idesc, s > 0);
          }
        }
      };
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        // conv0: T tiles of 128 rows (8 samples x 16 rows), gathered by the compute warps
        int T;
        if constexpr (S::kK0Chunks == 4) {  // f32 modes: per-K-chunk readiness
          mbar_wait(&bar_a0c[0], n_a0 & 1);
          T = s_T;  // written before the first chunk-0 arrival of this item
          mbar_wait(&bar_w[0], it & 1);
          tc_fence_after();
          for (int t = 0; t < T; ++t, ++n_a0) {
            for (int c = 0; c < 4; ++c) {
              if (t > 0 || c > 0) {
                mbar_wait(&bar_a0c[c], n_a0 & 1);
                tc_fence_after();
              }
              for (int s = 4 * c; s < 4 * c + 4 && s < S::kK0Steps; ++s) {
                const uint32_t ao = c * S::kStage + (s & 3) * 32, wo = c * S::kWChunk + (s & 3) * 32;
                const uint64_t ad = smem_desc_sw128(r1 + ao), bd = smem_desc_sw128(r2 + wo);
                const uint32_t d = tmem + t * S::kAccW;
                if (S::kSplit) {
                  mma<kMode>(d, ad, bd, idesc2, s > 0);
                  mma<kMode>(d + kC, smem_desc_sw128(r1 + S::kA0Lo + ao), bd, idesc, 1);
                } else {
                  mma<kMode>(d, ad, bd, idesc, s > 0);
                }
              }
            }
            mma_commit(&bar_t0);
          }
        } else {
          mbar_wait(&bar_a0, n_a0++ & 1);
          T = s_T;  // written before the first bar_a0 arrival of this item
          mbar_wait(&bar_w[0], it & 1);
          tc_fence_after();
          for (int t = 0; t < T; ++t) {
            if (t > 0) {
              mbar_wait(&bar_a0, n_a0++ & 1);
              tc_fence_after();
            }
            gemm(tmem + t * S::kAccW, S::kA0Lo, S::kK0Steps);
            mma_commit(&bar_t0);
          }
        }
        mma_commit(&bar_c0);
        // conv1: two tiles (16 positions x 8 samples each), A restaged by the
        // epilogue; tile 1 is all-constant (skipped) when every context fits in tiles 0-1
        const int n_c1 = (T <= 2 && p.c1acc) ? 1 : 2;
        for (int u = 0; u < n_c1; ++u) {
          mbar_wait(&bar_a1, n_a1++ & 1);
          if (u == 0) mbar_wait(&bar_w[1], it & 1);
          tc_fence_after();
          gemm(tmem + S::kConv1Col + u * S::kAccW, S::kALo, 4 * S::kKChunks);
          mma_commit(&bar_m1);
        }
        mma_commit(&bar_w1f);
        // conv2: one tile of 128 rows (8 samples x 16 positions)
        mbar_wait(&bar_a2, it & 1);
        mbar_wait(&bar_w[2], it & 1);
        tc_fence_after();
        gemm(tmem + S::kConv2Col, S::kALo, 4 * S::kKChunks);
        mma_commit(&bar_m2);
      }
    }
    __syncwarp();
  } else {
    // ---------------- compute warps 0-7 ----------------
    const int tid = threadIdx.x;  // 0..255
    const int quad = warp & 3, half = warp >> 2;
    const int m = quad * 32 + lane;  // TMEM lane owned by this thread
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const k1::ApplyArgs aa{p.bw, p.max_context, p.per_cycle, 1, p.iflags, p.nc};
    const NormConsts& nc = *p.nc;
    uint32_t n_t0 = 0, n_m1 = 0;
    int it = 0;
    long long* tr = p.trace ? p.trace + blockIdx.x * 32 : nullptr;
    // extra per-warp-0 stamps of the first item (no barrier: warp 0's own progress)
    long long* tx = p.trace ? p.trace + kChainTraceFrontX + blockIdx.x * 16 : nullptr;
    auto stampx = [&](int i) {
      if (tx && it == 0 && tid == 0) tx[i] = clock64();
    };
    // diagnostics: phase-boundary clocks of the first item, taken after a
    // barrier of the compute warps so a mark means "all of them are done"
    auto mark = [&](int i) {
      if (tr && it == 0) {
        compute_sync();
        if (tid == 0) tr[i] = clock64();
      }
    };
    mark(0);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // SubState / rings of the previous round
    if (tr && tid == 0) tr[15] = clock64();
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      // ---- 1. decode the previous round (FC tail of the item's 8 samples, all
      //         warps), then apply + column table: warp w owns sub-trace item*8 + w ----
      {
        const uint64_t s = p.first + static_cast<uint64_t>(item) * kItem + warp;
        const bool mine = s < p.last && !p.calibrate;
        // R1 is idle until the gather: W2 (bulk copy) | h [8][hidden] | y [8][64]
        if (tr && it == 0 && lane == 0 && warp == 0) tr[24] = clock64();
        float* hs = reinterpret_cast<float*>(R1) + kFcMaxOut * kFcMaxHidden;
        float* ys = hs + kItem * kFcMaxHidden;
        cta8_fc(p.fc, (mine ? s : p.first) - p.first, reinterpret_cast<const float*>(R1), hs, ys,
                (tr && it == 0) ? tr + 28 : nullptr, &bar_w2, it & 1,
                kMulti && it > 0 ? reinterpret_cast<const float*>(R2) : nullptr, &bar_part, &bar_pread, (it - 1) & 1);
        if (tr && it == 0 && lane == 0 && warp == 0) tr[25] = clock64();
        int ncs = -1;
        if (mine) {
          const k1::Rings r = k1::rings_of(p.proc, p.wq, p.pmask, p.wmask, s);
          SubState* sp = p.state + s;
          mbar_wait(&bar_st, it & 1);  // prefetched by the producer during the decode
          SubState st = s_state[warp];
          bool dirty = false;
          if (st.status == kOk && st.awaiting) {  // K3 of the previous round for this sub-trace
            uint32_t tri[3];
            warp_decode_triple(ys + warp * kFcMaxOut, s_lab, p.fc.class_fetch, p.fc.class_exec, p.fc.class_store,
                               (st.t_flags & kFlagStore) != 0, tri);
            if (tr && it == 0 && lane == 0 && warp == 0) tr[26] = clock64();
            apply_decoded_reg(st, tri, p.fc.pred_fetch, p.per_cycle);
            st.awaiting = 0;
            dirty = true;
          }
          if (st.status == kOk && st.has_pend) {
            k1::apply_step(st, r, aa);
            dirty = true;
          }
          if (tr && it == 0 && lane == 0 && warp == 0) tr[27] = clock64();
          if (dirty) {
            if (lane == 0) *sp = st;
            __syncwarp();
          }
          if (tr && it == 0 && lane == 0) tr[16 + warp] = clock64();  // per-warp apply done
          if (st.status == kOk && st.pos < st.len) {
            const uint64_t tgt = st.begin + st.pos;
            const uint32_t ncols = min(static_cast<uint32_t>(p.max_context), (st.pt - st.ph) + (st.wt - st.wh));
            stampx(5);
            mbar_wait(&bar_tg, it & 1);
            stampx(6);
            const bool pre = s_tidx[warp] == tgt;  // the producer's prediction of this round's target
            const uint64_t tpc = pre ? s_tpc[warp] : p.pc[tgt];
            const uint64_t taddr = pre ? s_taddr[warp] : p.addr[tgt];
            const uint8_t tfl = pre ? static_cast<uint8_t>(s_tfl[warp]) : p.iflags[tgt];
            const bool tmemop = (tfl & kFlagMem) != 0;
            uint32_t* ti = tbl_inst + warp * kTblCols;
            float4* td = tbl_dyn + warp * kTblCols;
            for (uint32_t c = lane; c <= ncols; c += 32) {
              if (c == 0) {
                ti[0] = static_cast<uint32_t>(tgt);
                td[0] = make_float4(s_zero[kSlotResidence], s_zero[kSlotExecution], s_zero[kSlotStore], 0.0f);
                continue;
              }
              const RingEntry e = k1::context_entry(st, r, c - 1);
              const int32_t res = static_cast<int32_t>(static_cast<uint32_t>(st.cur - e.push));
              const uint32_t f = k1::dep_flags(tpc, taddr, tmemop, e, p.line, p.page);
              ti[c] = static_cast<uint32_t>(st.begin + e.idx);
              td[c] = make_float4(norm_slot(res, nc.mean[kSlotResidence], nc.sd[kSlotResidence]), e.nexec, e.nstore,
                                  __uint_as_float(f));
            }
            stampx(7);
            if (lane == 0) {  // the next round's push carries these into the ring entry
              sp->awaiting = 1;
              sp->xcols = ncols + 1;
              sp->t_pc = tpc;
              sp->t_addr = taddr;
              sp->t_flags = tfl;
            }
            ncs = static_cast<int>(ncols);
          }
        }
        if (lane == 0) s_ncols[warp] = ncs;
      }
      compute_sync();
      mark(1);
      int T = 1;  // conv0 tiles with any non-zero row (rows of 2 columns: ceil((ncols + 1) / 2))
#pragma unroll
      for (int w = 0; w < kItem; ++w) {
        const int rows = (s_ncols[w] + 2) >> 1;
        T = max(T, (rows + kRowsT - 1) / kRowsT);
      }
      if (tid == 0) s_T = T;

      // ---- 2. gather conv0 tiles straight into the A operand ----
      // Thread = (sample `warp`, column 32t + lane): one A half-row (50 slots of
      // one context column) per thread per tile: 11 float4 static-slot loads in
      // flight, the 9 dynamic slots from the column table, 16-B stores.
      mbar_wait(&bar_stg, it & 1);  // tile-0 staging landed (issued by the producer during the decode)
      const long long t_gather0 = tx ? clock64() : 0;
      if (tx && it == 0 && tid == 0) tx[10] = t_gather0;
      for (int t = 0; t < T; ++t) {
        // lane -> (position q of the tile, K half h); row slot: even positions
        // in slots 0-7, odd in 8-15 (see row_slot_c0 below)
        const int q = 2 * ((lane >> 1) & 7) + (lane >> 4), h = lane & 1;
        const int col = 32 * t + 2 * q + h;
        const int r = warp * kRowsT + (lane >> 4) * 8 + ((lane >> 1) & 7);
        const bool live = col <= s_ncols[warp];
        float v[kSlots];
        {
          // the row's 41 static slots: six 32-B loads (one L2 sector each; rows
          // are 192 B, sector aligned) instead of eleven 16-B ones
          const uint32_t row = live ? tbl_inst[warp * kTblCols + col] : 0u;
          const float* srow = p.stat + static_cast<uint64_t>(row) * kStatStride;
          const uint32_t slo = s_stg_lo[warp], shi = s_stg_hi[warp];
          const bool staged = t == 0 && live && row >= slo && row <= shi;
          float w[48];
#pragma unroll
          for (int i = 0; i < 48; ++i) w[i] = 0.0f;
          if (staged) {  // from the R1 staging (landed during the decode)
            const float4* sp = reinterpret_cast<const float4*>(R1 + kStgOff + warp * kStgBox + (row - slo) * kStgPitch);
#pragma unroll
            for (int i = 0; i < 11; ++i) {
              const float4 x = sp[i];
              w[4 * i] = x.x;
              w[4 * i + 1] = x.y;
              w[4 * i + 2] = x.z;
              w[4 * i + 3] = x.w;
            }
          } else if (live) {
#pragma unroll
            for (int i = 0; i < 6; ++i)
              asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                           : "=f"(w[8 * i]), "=f"(w[8 * i + 1]), "=f"(w[8 * i + 2]), "=f"(w[8 * i + 3]),
                             "=f"(w[8 * i + 4]), "=f"(w[8 * i + 5]), "=f"(w[8 * i + 6]), "=f"(w[8 * i + 7])
                           : "l"(srow + 8 * i));
          }
#pragma unroll
          for (int i = 0; i <= 40; ++i) v[i] = w[i];
          const float4 d = tbl_dyn[warp * kTblCols + (live ? col : 0)];
          const uint32_t f = __float_as_uint(d.w);
          v[kSlotResidence] = d.x;
          v[kSlotExecution] = d.y;
          v[kSlotStore] = d.z;
#pragma unroll
          for (int b2 = 0; b2 < 5; ++b2)
            v[kSlotFlag0 + b2] = ((f >> b2) & 1u) ? s_one[kSlotFlag0 + b2] : s_zero[kSlotFlag0 + b2];
          v[kSlotReserved] = s_zero[kSlotReserved];
          if (!live) {
#pragma unroll
            for (int k = 0; k < kSlots; ++k) v[k] = 0.0f;
          }
        }
        if (tx && it == 0) {  // diagnostics: force the loads before the stamp
          float sum = 0.0f;
#pragma unroll
          for (int k = 0; k < kSlots; ++k) sum += v[k];
          if (sum == 12345.0f) tx[15] = 1;
          stampx(t == 0 ? 0 : 2);
          if (t == 0 && warp == 0) {  // per-lane completion spread of warp 0 (vs tx[10])
            const uint32_t now = static_cast<uint32_t>(clock64() - t_gather0);
            const uint32_t mn = __reduce_min_sync(0xffffffffu, now), mx = __reduce_max_sync(0xffffffffu, now);
            const uint32_t l1 = __shfl_sync(0xffffffffu, now, 2);
            if (lane == 0) {
              tx[8] = t_gather0 + mn;
              tx[9] = t_gather0 + mx;
              tx[11] = t_gather0 + l1;
            }
          }
        }
        // loads and values above overlap the previous tile's MMAs; only the
        // operand writes wait for them to finish reading R1 (tile 0: for every
        // thread to finish reading the staging, which the operand overlaps)
        if (t > 0) mbar_wait(&bar_t0, n_t0++ & 1);
        auto chunk_done = [&](int c) {  // this thread's part of K range [32c, 32c + 32) is written
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&bar_a0c[c]);
        };
        if constexpr (S::kK0Chunks == 4) {
          if (h == 0) {  // K 0-31 (chunk 0) first: it does not overlap the tile-0 staging
#pragma unroll
            for (int i = 0; i < 8; ++i) put4<kMode>(R1, S::kA0Lo, r, 4 * i, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            chunk_done(0);
          }
        }
        // 3xTF32: the lo planes of chunks 1-3 overlap the staging, so tile 0
        // waits for every thread to have read its staged rows (bf16 / fp8
        // operands end below the staging: no wait)
        if (S::kSplit && t == 0) compute_sync();
        if (t == 1) stampx(3);
        if constexpr (S::kK0Chunks == 4) {
          if (h == 0) {  // the rest of K 0..49: its part of chunk 1
#pragma unroll
            for (int i = 8; i < 12; ++i) put4<kMode>(R1, S::kA0Lo, r, 4 * i, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            put2<kMode>(R1, S::kA0Lo, r, 48, v[48], v[49]);
            chunk_done(1);
          } else {  // K 50..99 + pad: its part of chunk 1 (K 50-63), chunk 2 (64-95), chunk 3 (96-103)
            put2<kMode>(R1, S::kA0Lo, r, 50, v[0], v[1]);
#pragma unroll
            for (int i = 0; i < 3; ++i)
              put4<kMode>(R1, S::kA0Lo, r, 52 + 4 * i, v[2 + 4 * i], v[3 + 4 * i], v[4 + 4 * i], v[5 + 4 * i]);
            chunk_done(1);
#pragma unroll
            for (int i = 3; i < 11; ++i)
              put4<kMode>(R1, S::kA0Lo, r, 52 + 4 * i, v[2 + 4 * i], v[3 + 4 * i], v[4 + 4 * i], v[5 + 4 * i]);
            chunk_done(2);
            put4<kMode>(R1, S::kA0Lo, r, 96, v[46], v[47], v[48], v[49]);
#pragma unroll
            for (int k = 100; k < 100 + 2 * S::kPadUnits; k += 2) put2<kMode>(R1, S::kA0Lo, r, k, 0.0f, 0.0f);
            chunk_done(3);
          }
        } else if (h == 0) {  // K 0..49
#pragma unroll
          for (int i = 0; i < 12; ++i) put4<kMode>(R1, S::kA0Lo, r, 4 * i, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          put2<kMode>(R1, S::kA0Lo, r, 48, v[48], v[49]);
        } else {  // K 50..99, then the zero pad up to the last k-step
          put2<kMode>(R1, S::kA0Lo, r, 50, v[0], v[1]);
#pragma unroll
          for (int i = 0; i < 12; ++i)
            put4<kMode>(R1, S::kA0Lo, r, 52 + 4 * i, v[2 + 4 * i], v[3 + 4 * i], v[4 + 4 * i], v[5 + 4 * i]);
#pragma unroll
          for (int k = 100; k < 100 + 2 * S::kPadUnits; k += 2) put2<kMode>(R1, S::kA0Lo, r, k, 0.0f, 0.0f);
        }
        if (p.dump) {
          const int row = t * kRowsT + q;
          const uint64_t smp = static_cast<uint64_t>(item) * kItem + warp;
          if (smp < samples && (row + 1) * 100 <= static_cast<int>(p.dump_stride)) {
            float* o = p.dump + smp * p.dump_stride + row * 100 + 50 * h;
#pragma unroll
            for (int k = 0; k < kSlots; k += 2) *reinterpret_cast<float2*>(o + k) = make_float2(v[k], v[k + 1]);
          }
        }
        stampx(t == 0 ? 1 : 4);
        if constexpr (S::kK0Chunks != 4) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&bar_a0);
        }
        mark(2 + t);
      }
      if (tr && it == 0 && tid == 0) tr[20] = T;
      // ---- 3. restage conv0 -> conv1 A (two tiles), conv1 -> conv2 A ----
      mbar_wait(&bar_t0, n_t0++ & 1);  // last conv0 tile done: all conv0 accumulators final, R1 free
      tc_fence_after();
      mark(6);
      const int n_c1 = (T <= 2 && p.c1acc) ? 1 : 2;  // same rule as the MMA warp
      for (int u = 0; u < n_c1; ++u) {
        if (u == 1) {
          mbar_wait(&bar_m1, n_m1++ & 1);  // conv1 tile 0 consumed R1
          tc_fence_after();
        }
        // conv0 tile t = 2u + half, row m = (sample m/16, slot m%16 = position
        // 16t + 2(m%8) + (m%16)/8) -> conv1 tile u, position 8*half + m%8, K half (m%16)/8
        const int t = 2 * u + half;
        restage_row<kMode>(R1, tmem + lane_off + t * S::kAccW, t >= T ? s_zacc : nullptr,
                           (m >> 4) * 16 + conv1_slot(8 * half + (m & 7)), ((m >> 3) & 1) * kC, sbias[0],
                           p.wscale[0]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&bar_a1);
        mark(7 + u);
      }
      mbar_wait(&bar_m1, n_m1++ & 1);  // last conv1 tile done
      tc_fence_after();
      mark(9);
      if (p.c1acc_out && item == 0 && warp == 0) {  // calibration: conv1 row (sample 0, position 0)
#pragma unroll 1
        for (int c0 = 0; c0 < kC; c0 += 16) {
          float v[16];
          tmem_ld16(tmem + lane_off + S::kConv1Col + c0, v);
          if constexpr (S::kSplit) {  // + the cross half
            float x[16];
            tmem_ld16(tmem + lane_off + S::kConv1Col + kC + c0, x);
            for (int i = 0; i < 16; ++i) v[i] += x[i];
          }
          if (lane == 0)
            for (int i = 0; i < 16; ++i) p.c1acc_out[c0 + i] = v[i];
        }
      }
      // conv1 tile `half`, row m = (sample m/16, slot m%16 holding position
      // 16*half + p, conv1_slot(p) = m%16) -> conv2 row (m/16)*16 + 8*half + p/2, K half p%2
      {
        const int sl = m & 15;
        const int pair = sl < 8 ? sl : ((sl & 7) ^ 4);  // p / 2
        restage_row<kMode>(R1, tmem + lane_off + S::kConv1Col + half * S::kAccW,
                           (half == 1 && n_c1 == 1) ? s_c1 : nullptr,
                           (m >> 4) * 16 + 8 * half + pair, (sl >> 3) * kC, sbias[1], p.wscale[1]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&bar_a2);
      mark(10);

      // ---- 4. conv2 -> flat[sample][pos*64 + c]: row m is flat row item*128 + m ----
      mbar_wait(&bar_m2, it & 1);
      tc_fence_after();
      mark(11);
      const uint64_t sample = static_cast<uint64_t>(item) * kItem + (m >> 4);
      const bool out_tma = kMode != kBF16 && p.out_tma;
      if (out_tma) {
        // stage the 32 columns of row m in R1 (idle after conv2: the next item's
        // W2 lands below 64 KB) as 128 rows x 128 B per column half, SWIZZLE_128B;
        // each warp TMA-stores its 32 x 32 box, rows past the batch clipped
        uint8_t* stg = R1 + kOutStage + half * S::kStage;
        float v[32];
        tmem_ld16(tmem + lane_off + S::kConv2Col + half * 32, v);
        tmem_ld16(tmem + lane_off + S::kConv2Col + half * 32 + 16, v + 16);
        if constexpr (S::kSplit) {  // + the cross half
          float x[32];
          tmem_ld16(tmem + lane_off + S::kConv2Col + kC + half * 32, x);
          tmem_ld16(tmem + lane_off + S::kConv2Col + kC + half * 32 + 16, x + 16);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += x[i];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stg + m * 128 + ((q ^ (m & 7)) << 4)) =
              make_float4(fmaxf(v[4 * q] + sbias[2][half * 32 + 4 * q], 0.0f),
                          fmaxf(v[4 * q + 1] + sbias[2][half * 32 + 4 * q + 1], 0.0f),
                          fmaxf(v[4 * q + 2] + sbias[2][half * 32 + 4 * q + 2], 0.0f),
                          fmaxf(v[4 * q + 3] + sbias[2][half * 32 + 4 * q + 3], 0.0f));
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmOut, stg + quad * 32 * 128, half * 32, item * (kItem * 16) + quad * 32);
          bulk_commit();
        }
      }
      for (int c0 = half * 32; c0 < half * 32 + 32 && !out_tma; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + lane_off + S::kConv2Col + c0, v);
        if constexpr (S::kSplit) {
          float x[16];
          tmem_ld16(tmem + lane_off + S::kConv2Col + kC + c0, x);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += x[i];
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if constexpr (kMode == kFP8) v[i] *= p.wscale[2];
          v[i] = fmaxf(v[i] + sbias[2][c0 + i], 0.0f);
        }
        if (sample < samples) {
          const uint64_t off = static_cast<uint64_t>(item) * (kItem * 16 * kC) + m * kC + c0;
          if constexpr (kMode == kFP8) {
            uint4 pk;
            uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              w[i] = static_cast<uint32_t>(fp8x2(v[4 * i], v[4 * i + 1])) |
                     (static_cast<uint32_t>(fp8x2(v[4 * i + 2], v[4 * i + 3])) << 16);
            *reinterpret_cast<uint4*>(static_cast<uint8_t*>(p.out) + off) = pk;
          } else if (kMode == kBF16) {
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
      if (lane == 0) {
        if (out_tma) bulk_wait_read();  // staging is read: R1 reusable
        mbar_arrive(&bar_fo);
      }
      compute_sync();  // TMEM conv2 columns and the tables are free for the next item
      mark(12);
    }
  }
  if (kMode != kBF16 && p.out_tma && warp < 8 && lane == 0) bulk_wait_all();  // flat stores complete
  tc_fence_before();
  __syncthreads();
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 32 + 14] = global_ns();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    if (p.trace && lane == 0) p.trace[blockIdx.x * 32 + 31] = global_ns();  // diagnostics: about to exit
  }
}

// One warp per sub-trace: decode the last outstanding prediction, apply it,
// drain (simcore.cpp:152-159).
__global__ void __launch_bounds__(256) final_decode_kernel(FrontParams p) {
  extern __shared__ __align__(16) float fin_sm[];  // W2 [od][hidden] | h [8][hidden] | y [8][64]
  __shared__ double s_lab[6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 6) s_lab[threadIdx.x] = threadIdx.x < 3 ? p.nc->label_mean[threadIdx.x] : p.nc->label_sd[threadIdx.x - 3];
  float* w2s = fin_sm;
  float* hs = fin_sm + p.fc.od * p.fc.hidden;
  float* ys = hs + 8 * p.fc.hidden;
  for (int i = threadIdx.x; i < p.fc.od * p.fc.hidden / 4; i += 256)
    reinterpret_cast<float4*>(w2s)[i] = __ldg(reinterpret_cast<const float4*>(p.fc.w2t) + i);
  __syncthreads();
  const uint64_t s = p.first + static_cast<uint64_t>(blockIdx.x) * 8 + warp;
  cta8_fc(p.fc, (s < p.last ? s : p.first) - p.first, w2s, hs, ys);
  if (s >= p.last) return;
  const k1::ApplyArgs aa{p.bw, p.max_context, p.per_cycle, 1, p.iflags, p.nc};
  const k1::Rings r = k1::rings_of(p.proc, p.wq, p.pmask, p.wmask, s);
  SubState* sp = p.state + s;
  SubState st = *sp;
  if (st.status == kOk && st.awaiting) {
    uint32_t tri[3];
    warp_decode_triple(ys + warp * kFcMaxOut, s_lab, p.fc.class_fetch, p.fc.class_exec, p.fc.class_store,
                       (st.t_flags & kFlagStore) != 0, tri);
    apply_decoded_reg(st, tri, p.fc.pred_fetch, p.per_cycle);
    st.awaiting = 0;
  }
  if (st.status == kOk && st.has_pend) k1::apply_step(st, r, aa);
  if (lane == 0) *sp = st;
}

void launch_final_decode(const FrontParams& p, cudaStream_t s) {
  const uint64_t n = p.last - p.first;
  if (n == 0) return;
  const size_t sm = (static_cast<size_t>(p.fc.od + 8) * p.fc.hidden + 8 * kFcMaxOut) * 4;
  if (sm > 48 * 1024)  // (od + 8) x hidden W2 / h staging: output_dim >= 39 at hidden 256
    CUDA_OK(cudaFuncSetAttribute(final_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sm)));
  final_decode_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, sm, s>>>(p);
}

namespace {
size_t front_smem_bytes() { return kR1 + kR2 + kTbl + 1024; }
}  // namespace

void launch_round_front(int mode, const CUtensorMap* w, const FrontParams& p, int num_sms, cudaStream_t s) {
  const uint64_t samples = p.last - p.first;
  if (samples == 0) return;
  if (p.max_context + 1 > kTblCols) throw ApiError("fused round front: max_context too large");
  const uint64_t items = (samples + kItem - 1) / kItem;
  const dim3 grid(static_cast<unsigned>(items < static_cast<uint64_t>(num_sms) ? items : num_sms));
  const size_t sm = front_smem_bytes();
  const bool multi = items > grid.x;
#define SIMNET_FRONT(M, MU) \
  launch_pdl_tag("front", round_front_kernel<M, MU>, grid, dim3(kThreadsRF), sm, s, w[0], w[1], w[2], w[3], w[4], \
                 w[5], w[6], w[7], p)
  if (mode == kFP8)
    multi ? SIMNET_FRONT(kFP8, true) : SIMNET_FRONT(kFP8, false);
  else if (mode == kBF16)
    multi ? SIMNET_FRONT(kBF16, true) : SIMNET_FRONT(kBF16, false);
  else if (mode == kTF32)
    multi ? SIMNET_FRONT(kTF32, true) : SIMNET_FRONT(kTF32, false);
  else
    multi ? SIMNET_FRONT(kTF32x3, true) : SIMNET_FRONT(kTF32x3, false);
#undef SIMNET_FRONT
}

void round_front_set_attributes() {
  const int sm = static_cast<int>(front_smem_bytes());
  CUDA_OK(cudaFuncSetAttribute(round_front_kernel<kBF16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(round_front_kernel<kTF32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(round_front_kernel<kTF32x3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(round_front_kernel<kBF16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(round_front_kernel<kFP8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(round_front_kernel<kFP8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(round_front_kernel<kTF32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  CUDA_OK(cudaFuncSetAttribute(round_front_kernel<kTF32x3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
}

}  // namespace simnet
