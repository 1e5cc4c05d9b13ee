// K2 on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Each conv layer of the reference CNN (cnn.cpp:90-125) is one GEMM over
// (sample, position) rows: out[m, n] = ReLU(sum_k A[m, k] W[n, k] + b[n]) with
// A the previous activation viewed as [rows/2 x 2C] (kernel-2/stride-2
// windows are adjacent rows, so no im2col).  FC1 is the same GEMM over
// [samples x flat] with split-K partials; FC2 + the FC1 epilogue run in a
// small fp32 tail kernel.
//
// One CTA computes one 128 x BN output tile:
//   warp 0      TMA producer: every K chunk of A (and W) into SWIZZLE_128B smem
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  (tf32x3) hi/lo operand split in smem; then the epilogue:
//               tcgen05.ld accumulator -> bias/ReLU -> global (f32 or bf16)
// Precisions: kind::f16 with bf16 operands; kind::tf32; 3xTF32 (A = hi + lo,
// W = hi + lo, D += Alo*Whi + Ahi*Wlo + Ahi*Whi, fp32-faithful).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <deque>
#include <vector>

#include "conv_chain.cuh"
#include "round_front.cuh"
#include "decode.cuh"
#include "tc_common.cuh"
#include "launch.cuh"
#include "model.cuh"
#include "sim_kernels.cuh"

namespace simnet {

// --------------------------------------------------------------------------
// Persistent, warp-specialised layer GEMM
// --------------------------------------------------------------------------
// CTA (gx, ny, nz) owns weight slice (N tile ny, K split nz), resident in smem
// for the whole launch, and loops over M tiles gx, gx + gridDim.x, ...
//   warp 0     TMA producer: A chunks (128 rows x 128 B) into a 4-stage ring
//   warp 1     TMEM allocation + single-thread tcgen05.mma issue
//   warps 2-5  (3xTF32) split each landed chunk into hi / lo in place
//   warps 6-9  epilogue: tcgen05.ld -> bias / ReLU -> global; two TMEM
//              accumulators so tile t's epilogue overlaps tile t+1's MMAs
constexpr int kStages = 4;     // default A ring depth
constexpr int kMaxStages = 6;  // CTAs looping over M tiles may trade a staging buffer for two more stages
constexpr int kWarps = 10;
constexpr int kLayerThreads = kWarps * 32;
constexpr uint32_t kAChunk = kBM * 128;  // 16 KB

struct TcGemmParams {
  int m;              // valid output rows
  int m_tiles;
  int n;              // BN: output columns per tile (multiple of 16, <= 128)
  int chunks;         // K chunks (128 B) per tile for this CTA's split
  int ksteps_last;    // MMA k-steps in the last chunk (1..4)
  int a3d;            // A map is 3-D (conv0 over the gathered input)
  int a_samples_box;  // 3-D: samples per 128-row box
  const float* bias;  // [n_total] (null: none)
  int relu;
  void* out;          // row-major [m][ldo] f32 or bf16
  int ldo;
  int out_bf16;
  uint64_t out_split_stride;  // elements between split-K partial planes
  long long* trace;           // diagnostics (SIMNET_CHAIN_TRACE): per-CTA event clocks, 16 per CTA
  int stages;                 // A ring depth (2..kStages; 0 = kStages)
  float out_scale;            // fp8: 1 / (power-of-two weight scale), applied to the accumulator
  int a_tmem;                 // 3xTF32: the split warps write A hi / lo into tensor memory (4-slot ring
                              // next to the accumulators) and the MMAs read A from there (SMEM: W only)
  int tma_out;                // f32 split-K partials through tmOut: CTAs owning one M tile stage the
                              // accumulator in the idle A ring and TMA-store it (coalesced, async)
  int gx_max;                 // CTAs per (N tile, K split) group along M (0 = as many as fit the SMs)
  int diag_skip_w;            // diagnostics (SIMNET_DIAG_FC1_SKIP_W, timing only: results are garbage):
                              // no weight loads, to measure their share of FC1
  int tma_multi;              // f32 split-K partials through tmOut for CTAs that loop over M tiles: two
                              // 16 KB staging buffers past the A ring, one 32-column group at a time
  int stg_bufs;               // tma_multi staging buffers (2, or 1 to make room for a deeper A ring)
  int diag_a_early;           // diagnostics (SIMNET_DIAG_FC1_A_EARLY, timing only: results are garbage):
                              // A loads issued without the dependency wait
  int stream_w;               // weights streamed through the ring with A (chunk by chunk, all of K in
                              // one CTA): no resident slice, no split-K planes (large-M conv layers)
};

template <int kMode, bool kAInTmem = false>
__global__ void __launch_bounds__(kLayerThreads, 1)
tc_layer_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ CUtensorMap tmOut,
                TcGemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  constexpr bool kSplit = kMode == kTF32x3;
  uint8_t* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
  const uint32_t bBytes = static_cast<uint32_t>(p.n) * 128;
  const bool sw = p.stream_w != 0;
  uint8_t* sW = base;                                      // [chunks][n x 128 B] (resident slice)
  uint8_t* sWlo = sW + (sw ? 0 : p.chunks * bBytes);       // tf32x3 only
  uint8_t* sA = sWlo + (kSplit && !sw ? p.chunks * bBytes : 0);  // [stages][16 KB]
  const int ns = p.stages > 0 ? p.stages : kStages;       // A ring depth
  uint8_t* sAlo = sA + ns * kAChunk;                       // tf32x3 only
  // tma_multi: 2 x 16 KB epilogue staging past the A ring (and its lo plane)
  uint8_t* sStg = sAlo + (kSplit && !kAInTmem ? ns * kAChunk : 0);
  // stream_w: the weight chunks ride in the ring, [stages][n x 128 B] (+ lo)
  uint8_t* sWr = sStg;
  uint8_t* sWrlo = sWr + ns * bBytes;

  __shared__ __align__(8) uint64_t bar_w;
  __shared__ __align__(8) uint64_t bar_full[kMaxStages], bar_split[kMaxStages], bar_empty[kMaxStages];
  __shared__ __align__(8) uint64_t bar_acc_full[2], bar_acc_empty[2];
  __shared__ __align__(8) uint64_t bar_sfree[kMaxStages], bar_tfree[4];  // a_tmem: SMEM stage read / TMEM A slot free
  __shared__ uint32_t tmem_slot;
  constexpr bool a_tmem = kSplit && kAInTmem;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntile = blockIdx.y, ks = blockIdx.z;
  const int kc0 = ks * p.chunks;  // first K chunk of this split
  const uint32_t tcols =
      a_tmem ? 512u : (2 * p.n <= 32 ? 32u : (2 * p.n <= 64 ? 64u : (2 * p.n <= 128 ? 128u : 256u)));
  constexpr uint32_t kATmem = 256;  // a_tmem: A ring columns [256, 512): slot g % 4 = hi 32 | lo 32

  if (threadIdx.x == 0) {
    mbar_init(&bar_w, 1);
    for (int i = 0; i < kMaxStages; ++i) {
      mbar_init(&bar_full[i], 1);
      mbar_init(&bar_split[i], 128);
      mbar_init(&bar_empty[i], 1);
      mbar_init(&bar_sfree[i], 128);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&bar_tfree[i], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_acc_full[i], 1);
      mbar_init(&bar_acc_empty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const uint32_t tmem = tmem_slot;
  const int elems = mode_chunk_elems(kMode);  // elements per 128 B chunk
  const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  long long* tr = p.trace ? p.trace + 148 * 32 + cta * 32 : nullptr;  // 32 words per CTA
  if (tr && threadIdx.x == 0) {
    tr[15] = 0;
    tr[0] = clock64();
    tr[8] = global_ns();
  }
  // PDL: let the next kernel start its prologue; everything above overlapped
  // the previous kernel.  Weights are constants and may be fetched before the
  // dependency wait; activations only after it.
  asm volatile("griddepcontrol.launch_dependents;");

  // A CTA that owns exactly one M tile has its split warps (2-5) idle once the
  // tile's chunks are split: they drain half of the accumulator columns.
  const bool solo = blockIdx.x < p.m_tiles && blockIdx.x + gridDim.x >= p.m_tiles && p.n % 32 == 0;
  const bool tma_out = solo && p.tma_out;
  // Solo CTA, TMA-stored partials: the tile's MMAs are done, so the A ring is
  // free; column group g (32 floats) of the accumulator goes to sA + g * 16 KB
  // as 128 rows x 128 B, SWIZZLE_128B (conflict-free 16-B stores), and each
  // warp TMA-stores its 32 rows x 32 columns boxes.
  auto epilogue_tma = [&](int t, int cb, int ce) {
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t tl = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const bool stamp = tr && warp == 6 && lane == 0;
    for (int c0 = cb; c0 < ce; c0 += 32) {
      float v[32];
      tmem_ld16(tl + c0, v);
      tmem_ld16(tl + c0 + 16, v + 16);
      if constexpr (kMode == kFP8) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= p.out_scale;
      }
      if (stamp && c0 == cb) tr[16] = clock64();  // first TMEM columns in registers
      uint8_t* stg = sA + (c0 >> 5) * kAChunk + r * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(stg + ((q ^ (r & 7)) << 4)) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      // this column group's box goes out while the next group is staged
      fence_async_smem();
      __syncwarp();
      if (lane == 0)
        tma_store_3d(&tmOut, sA + (c0 >> 5) * kAChunk + quad * 32 * 128, ntile * p.n + c0, t * kBM + quad * 32, ks);
    }
    if (stamp) tr[17] = clock64();  // staged
    if (stamp) tr[18] = clock64();  // fenced
    if (lane == 0) {
      bulk_commit();
      if (stamp) tr[19] = clock64();  // stores issued
      bulk_wait_read();  // staging read; the stores complete with the grid (dependents wait for it)
      if (stamp) tr[20] = clock64();  // staging read back
    }
  };
  // CTAs looping over M tiles: accumulator `acc` of tile t, 32-column groups
  // staged alternately in the two staging buffers (each warp its own 32 rows
  // x 128 B, SWIZZLE_128B) and TMA-stored, instead of per-thread row stores
  // (each of those touches 32 lines per instruction).  `ng` counts this
  // warp's groups, so a buffer is rewritten only after the store issued two
  // groups earlier has read it.
  auto epilogue_tma_multi = [&](int t, int acc, uint32_t& ng) {
    const int quad = warp & 3;
    const uint32_t tl = tmem + (static_cast<uint32_t>(quad * 32) << 16) + acc * p.n;
    for (int c0 = 0; c0 < p.n; c0 += 32, ++ng) {
      float v[32];
      tmem_ld16(tl + c0, v);
      tmem_ld16(tl + c0 + 16, v + 16);
      if constexpr (kMode == kFP8) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= p.out_scale;
      }
      const bool one = p.stg_bufs == 1;
      uint8_t* box = sStg + (one ? 0u : (ng & 1u)) * kAChunk + quad * 32 * 128;
      if (lane == 0) {  // the store that last used this buffer has read it
        if (one && ng >= 1) bulk_wait_read();
        if (!one && ng >= 2) bulk_wait_read1();
      }
      __syncwarp();
      uint8_t* stg = box + lane * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(stg + ((q ^ (lane & 7)) << 4)) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(&tmOut, box, ntile * p.n + c0, t * kBM + quad * 32, ks);
        bulk_commit();
      }
    }
  };
  auto epilogue = [&](int t, int acc, int cb, int ce) {
    const int quad = warp & 3;
    const int row = t * kBM + quad * 32 + lane;
    const uint32_t tl = tmem + (static_cast<uint32_t>(quad * 32) << 16) + acc * p.n;
    for (int c0 = cb; c0 < ce; c0 += 16) {
      float v[16];
      tmem_ld16(tl + c0, v);
      if constexpr (kMode == kFP8) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= p.out_scale;
      }
      if (row < p.m) {
        const int col = ntile * p.n + c0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (p.bias) v[i] += p.bias[col + i];
          if (p.relu) v[i] = fmaxf(v[i], 0.0f);
        }
        if (p.out_bf16) {
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + static_cast<uint64_t>(row) * p.ldo + col;
          uint4 pk[2];
          uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t*>(&b2);
          }
          reinterpret_cast<uint4*>(o)[0] = pk[0];
          reinterpret_cast<uint4*>(o)[1] = pk[1];
        } else {
          float* o = static_cast<float*>(p.out) + ks * p.out_split_stride + static_cast<uint64_t>(row) * p.ldo + col;
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
      }
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      // resident weights for this CTA's (N tile, K split)
      if (p.diag_skip_w || sw) {
        mbar_arrive(&bar_w);
      } else {
        mbar_expect_tx(&bar_w, p.chunks * bBytes * (kSplit ? 2u : 1u));
        for (int c = 0; c < p.chunks; ++c) {
          tma_load_2d(sW + c * bBytes, &tmB, &bar_w, (kc0 + c) * elems, ntile * p.n);
          if (kSplit) tma_load_2d(sWlo + c * bBytes, &tmBlo, &bar_w, (kc0 + c) * elems, ntile * p.n);
        }
      }
      if (!p.diag_a_early) asm volatile("griddepcontrol.wait;" ::: "memory");
      if (tr) tr[12] = global_ns();  // the previous kernel's results are visible
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.m_tiles; t += gridDim.x) {
        for (int c = 0; c < p.chunks; ++c) {
          mbar_wait(a_tmem ? &bar_sfree[stage] : &bar_empty[stage], phase ^ 1);
          if (a_tmem && sw) mbar_wait(&bar_empty[stage], phase ^ 1);  // the stage's W chunk: MMAs done
          mbar_expect_tx(&bar_full[stage], kAChunk + (sw ? bBytes * (kSplit ? 2u : 1u) : 0u));
          const int kx = (kc0 + c) * elems;
          if (p.a3d)
            tma_load_3d(sA + stage * kAChunk, &tmA, &bar_full[stage], kx, 0, t * p.a_samples_box);
          else
            tma_load_2d(sA + stage * kAChunk, &tmA, &bar_full[stage], kx, t * kBM);
          if (sw) {  // this chunk's weights with it (released with the stage)
            tma_load_2d(sWr + stage * bBytes, &tmB, &bar_full[stage], kx, ntile * p.n);
            if (kSplit) tma_load_2d(sWrlo + stage * bBytes, &tmBlo, &bar_full[stage], kx, ntile * p.n);
          }
          if (++stage == ns) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp runs the loop (warp-uniform operands) and the
    // *_w forms elect the issuing thread inside the asm (tc_common.cuh)
    const bool t0 = tr && lane == 0;
    {
      mbar_wait(&bar_w, 0);
      __syncwarp();
      if (t0) tr[1] = clock64();
      const uint32_t idesc = instr_desc(mode_fmt(kMode), p.n);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      uint32_t g = 0;  // chunk counter (a_tmem: TMEM slot g % 4)
      for (int t = blockIdx.x; t < p.m_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&bar_acc_empty[acc], acc_phase ^ 1);
        __syncwarp();
        tc_fence_after();
        const uint32_t d = tmem + acc * p.n;
        for (int c = 0; c < p.chunks; ++c) {
          mbar_wait(kSplit ? &bar_split[stage] : &bar_full[stage], phase);
          __syncwarp();
          if (t0 && it == 0 && c < 4) tr[c == 0 ? 2 : 4 + c] = clock64();  // chunk c ready (5, 6, 7: chunks 1-3)
          tc_fence_after();
          const int steps = c == p.chunks - 1 ? p.ksteps_last : 4;
          const long long t_issue = tr ? clock64() : 0;
          if constexpr (a_tmem) {  // A hi / lo in TMEM slot g % 4 (columns: hi 32 | lo 32), W from SMEM
            const uint32_t slot = tmem + kATmem + (g & 3u) * 64u;
            for (int j = 0; j < steps; ++j) {
              const uint32_t boff = (sw ? stage : c) * bBytes + j * 32;  // stream_w: the stage's W chunk
              const uint64_t bd = smem_desc_sw128(su32(sw ? sWr : sW) + boff);
              const uint32_t first = (c == 0 && j == 0) ? 0u : 1u;
              mma_ts_w<kMode>(d, slot + 32 + j * 8, bd, idesc, first);  // small terms first
              mma_ts_w<kMode>(d, slot + j * 8, smem_desc_sw128(su32(sw ? sWrlo : sWlo) + boff), idesc, 1);
              mma_ts_w<kMode>(d, slot + j * 8, bd, idesc, 1);
            }
            mma_commit_w(&bar_tfree[g & 3u]);  // the TMEM slot is free once these MMAs retire
          }
          for (int j = 0; j < steps && !a_tmem; ++j) {
            const uint32_t aoff = stage * kAChunk + j * 32;
            const uint32_t boff = (sw ? stage : c) * bBytes + j * 32;
            const uint64_t ad = smem_desc_sw128(su32(sA) + aoff);
            const uint64_t bd = smem_desc_sw128(su32(sw ? sWr : sW) + boff);
            const uint32_t first = (c == 0 && j == 0) ? 0u : 1u;
            if (kSplit) {
              mma_w<kMode>(d, smem_desc_sw128(su32(sAlo) + aoff), bd, idesc, first);  // small terms first
              mma_w<kMode>(d, ad, smem_desc_sw128(su32(sw ? sWrlo : sWlo) + boff), idesc, 1);
              mma_w<kMode>(d, ad, bd, idesc, 1);
            } else {
              mma_w<kMode>(d, ad, bd, idesc, first);
            }
          }
          if (!a_tmem || sw) mma_commit_w(&bar_empty[stage]);  // the stage is free once these MMAs retire
          ++g;
          if (t0 && it == 0) tr[15] += clock64() - t_issue;  // diagnostics: cycles spent issuing
          if (++stage == ns) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_w(&bar_acc_full[acc]);
        if (t0 && it < 1) tr[3] = clock64();
        if (t0 && it < 8) tr[21 + it] = clock64();  // diagnostics: tile it's MMAs all issued
      }
    }
    __syncwarp();
  } else if (warp < 6) {
    if constexpr (a_tmem) {  // hi / lo split of each landed A chunk straight into TMEM: thread = A row
      const int quad = warp & 3;
      const int r = quad * 32 + lane;
      const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
      int stage = 0;
      uint32_t phase = 0;
      uint32_t g = 0;
      const bool st0 = tr && threadIdx.x == 64;  // diagnostics: split of chunks 0 / 1 (first tile)
      for (int t = blockIdx.x; t < p.m_tiles; t += gridDim.x) {
        for (int c = 0; c < p.chunks; ++c, ++g) {
          mbar_wait(&bar_full[stage], phase);
          if (st0 && g < 2) tr[g == 0 ? 11 : 30] = clock64();  // chunk 0 / 1 landed
          if (g >= 4) mbar_wait(&bar_tfree[g & 3u], ((g >> 2) - 1) & 1u);  // chunk g-4's MMAs done
          tc_fence_after();
          const uint8_t* row = sA + stage * kAChunk + r * 128;
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint4 u = *reinterpret_cast<const uint4*>(row + ((q ^ (r & 7)) << 4));
            const uint32_t x[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              // hi = x rounded to tf32 (cvt.rna); lo = x - hi, exact in fp32, read at tf32
              hi[4 * q + e] = (x[e] + 0x1000u) & 0xffffe000u;
              lo[4 * q + e] = __float_as_uint(__uint_as_float(x[e]) - __uint_as_float(hi[4 * q + e]));
            }
          }
          const uint32_t slot = tmem + lane_off + kATmem + (g & 3u) * 64u;
          tmem_st32(slot, hi);
          tmem_st32(slot + 32, lo);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bar_sfree[stage]);  // SMEM stage read
          mbar_arrive(&bar_split[stage]);  // TMEM slot written
          if (st0 && g < 2) tr[g == 0 ? 29 : 31] = clock64();  // chunk 0 / 1 split into TMEM
          if (++stage == ns) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    } else if (kSplit) {  // hi/lo split of each landed A chunk
      const int t128 = threadIdx.x - 64;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.m_tiles; t += gridDim.x) {
        for (int c = 0; c < p.chunks; ++c) {
          mbar_wait(&bar_full[stage], phase);
          float4* a = reinterpret_cast<float4*>(sA + stage * kAChunk);
          float4* alo = reinterpret_cast<float4*>(sAlo + stage * kAChunk);
#pragma unroll 4
          for (int i = t128; i < static_cast<int>(kAChunk / 16); i += 128) {
            const uint4 u = reinterpret_cast<const uint4*>(a)[i];
            // hi = x rounded to tf32 (round half away, cvt.rna); lo = x - hi is
            // exact in fp32 and is read by the MMA at tf32 precision
            uint4 h;
            h.x = (u.x + 0x1000u) & 0xffffe000u;
            h.y = (u.y + 0x1000u) & 0xffffe000u;
            h.z = (u.z + 0x1000u) & 0xffffe000u;
            h.w = (u.w + 0x1000u) & 0xffffe000u;
            float4 l;
            l.x = __uint_as_float(u.x) - __uint_as_float(h.x);
            l.y = __uint_as_float(u.y) - __uint_as_float(h.y);
            l.z = __uint_as_float(u.z) - __uint_as_float(h.z);
            l.w = __uint_as_float(u.w) - __uint_as_float(h.w);
            reinterpret_cast<uint4*>(a)[i] = h;
            alo[i] = l;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&bar_split[stage]);
          if (++stage == ns) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    if (solo) {  // second half of the single tile's accumulator columns
      asm volatile("griddepcontrol.wait;" ::: "memory");
      mbar_wait(&bar_acc_full[0], 0);
      tc_fence_after();
      if (tma_out)
        epilogue_tma(blockIdx.x, p.n / 2, p.n);
      else
        epilogue(blockIdx.x, 0, p.n / 2, p.n);
      tc_fence_before();
    }
  } else {
    // epilogue warps 6..9: TMEM lane quadrant = warp % 4
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int it = 0;
    uint32_t ng = 0;
    const bool multi_tma = !solo && p.tma_multi;
    for (int t = blockIdx.x; t < p.m_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      mbar_wait(&bar_acc_full[acc], (it >> 1) & 1);
      tc_fence_after();
      if (tr && warp == 6 && lane == 0 && it == 0) tr[14] = clock64();  // accumulator complete
      if (tma_out)
        epilogue_tma(t, 0, p.n / 2);
      else if (multi_tma)
        epilogue_tma_multi(t, acc, ng);
      else
        epilogue(t, acc, 0, solo ? p.n / 2 : p.n);
      tc_fence_before();
      mbar_arrive(&bar_acc_empty[acc]);
      if (tr && warp == 6 && lane == 0 && it < 1) {
        tr[4] = clock64();
        tr[10] = global_ns();
      }
    }
    if (multi_tma && lane == 0) bulk_wait_read();  // staging read (the stores complete with the grid)
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    // diagnostics: past the final barrier (thread 0, the producer lane, may
    // leave it before the epilogue warps arrive, so warp 1 takes the stamp)
    if (tr && lane == 0) tr[9] = global_ns();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
    if (tr && lane == 0) tr[13] = global_ns();  // diagnostics: TMEM released, CTA about to exit
  }
}

// FC tail (+ fused K3): 8 samples per block through cta8_fc (fc_decode.cuh:
// split-K reduction, ReLU, FC2 in a fixed batch-independent order), then,
// when simulating, the hybrid decode and clock advance of K3 per sample.
constexpr int kTailWarps = 8;
constexpr int kTailThreads = 32 * kTailWarps;
constexpr int kMaxSplit = kFcMaxSplit;  // split-K planes of FC1 (flat 1024 f32 = 32 chunks / 4)
constexpr int kMaxOut = kFcMaxOut;

struct TailParams {
  FcDecodeArgs fc;
  float* y;
  int samples;
  DecodeParams dec;  // dec.state == nullptr: outputs only
};

// dynamic smem: W2 [od][hidden] | h [kTailWarps][hidden] | y [kTailWarps][kMaxOut]
__global__ void __launch_bounds__(kTailThreads) fc_tail_kernel(TailParams p) {
  extern __shared__ __align__(16) float tail_sm[];
  __shared__ double s_lab[6];
  const int hid = p.fc.hidden, od = p.fc.od;
  if (threadIdx.x < 6 && p.dec.nc)
    s_lab[threadIdx.x] = threadIdx.x < 3 ? p.dec.nc->label_mean[threadIdx.x] : p.dec.nc->label_sd[threadIdx.x - 3];
  float* w2s = tail_sm;
  float* hs = w2s + od * hid;
  float* ys = hs + kTailWarps * hid;
  asm volatile("griddepcontrol.launch_dependents;");
  {  // W2 (a constant) is staged before the dependency wait
    const int total = od * hid / 4;
    const float4* src = reinterpret_cast<const float4*>(p.fc.w2t);
    for (int i = threadIdx.x; i < total; i += kTailThreads) reinterpret_cast<float4*>(w2s)[i] = __ldg(src + i);
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * kTailWarps + warp;
  cta8_fc(p.fc, static_cast<uint64_t>(s < p.samples ? s : 0), w2s, hs, ys);  // all 8 warps take part
  if (s >= p.samples) return;
  const float* y = ys + warp * kMaxOut;
  for (int o = lane; o < od; o += 32) p.y[static_cast<uint64_t>(s) * od + o] = y[o];
  SubState* sp = p.dec.state ? p.dec.state + p.dec.first + s : nullptr;
  if (sp && sp->status == kOk && sp->pos < sp->len) {
    uint32_t t[3];
    warp_decode_triple(y, s_lab, p.fc.class_fetch, p.fc.class_exec, p.fc.class_store,
                       (p.dec.iflags[sp->begin + sp->pos] & kFlagStore) != 0, t);
    if (lane == 0) apply_decoded(sp, t, p.dec.pred_fetch, p.dec.per_cycle);
  }
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw ApiError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// f32, no swizzle (byte-exact rows in shared memory)
CUtensorMap make_map_plain(const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                           const uint32_t* box) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t gd[3];
  cuuint64_t gs[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(ptr), gd, gs, bx, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ApiError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

// element size -> tensor-map data type (1: fp8 e4m3 as bytes, 2: bf16, 4: f32)
CUtensorMap make_map_e(const void* ptr, int esz, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t gd[3];
  cuuint64_t gs[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
  const CUtensorMapDataType dt = esz == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                          : (esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  const CUresult r = encode_fn()(&m, dt, rank, const_cast<void*>(ptr), gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ApiError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

CUtensorMap make_map(const void* ptr, bool bf16, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t gd[3];
  cuuint64_t gs[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
  const CUresult r = encode_fn()(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 rank, const_cast<void*>(ptr), gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ApiError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

float tf32_round_host(float x) {  // cvt.rna.tf32.f32: round half away from zero to 10 mantissa bits
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return x;
  u += 0x1000u;
  u &= 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// float -> fp8 e4m3 (round to nearest even, saturate to +-448; NaN -> 0x7f)
uint8_t fp8_e4m3_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  const uint8_t sign = static_cast<uint8_t>((u >> 24) & 0x80u);
  const float a = std::fabs(x);
  if (std::isnan(x)) return 0x7f;
  if (a >= 448.0f) return sign | 0x7e;  // max finite (satfinite)
  if (a < std::ldexp(1.0f, -10)) return sign;  // below half the smallest subnormal (2^-9): 0
  int e;
  std::frexp(a, &e);  // a = f * 2^e, f in [0.5, 1)
  int exp = e - 1;    // a = 1.xxx * 2^exp
  if (exp < -6) {     // subnormal: multiples of 2^-9
    const float q = std::nearbyint(std::ldexp(a, 9));  // round half even (default mode)
    const int m = static_cast<int>(q);
    if (m >= 8) return sign | 0x08;  // rounds up to the smallest normal
    return sign | static_cast<uint8_t>(m);
  }
  float mant = std::ldexp(a, -exp) - 1.0f;                       // [0, 1)
  int m = static_cast<int>(std::nearbyint(std::ldexp(mant, 3)));  // 3 bits, round half even
  if (m == 8) {
    m = 0;
    ++exp;
  }
  if (exp > 8 || (exp == 8 && m == 7)) return sign | 0x7e;
  return sign | static_cast<uint8_t>(((exp + 7) << 3) | m);
}

uint16_t bf16_rn_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(u >> 16);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

struct TcWeights {
  DevBuf hi, lo;  // K-major [npad][kpad] (f32, bf16 or fp8 e4m3)
  int n = 0, npad = 0, k = 0, kpad = 0, n_tile = 0;
  float inv_scale = 1.0f;  // fp8: weights are stored x 2^e; accumulators are multiplied back by 2^-e
  CUtensorMap map_hi{}, map_lo{};  // box: one 128-B K chunk x n_tile rows
};

int mode_of(int precision) {
  if (precision == ILSIM_PREC_FP8) return kFP8;
  return precision == ILSIM_PREC_BF16 ? kBF16 : (precision == ILSIM_PREC_TF32 ? kTF32 : kTF32x3);
}

}  // namespace

struct TcModel {
  int mode = kTF32x3;
  bool chain = false;  // C3 shape: fused conv chain kernel
  std::deque<TcWeights> conv;
  TcWeights fc1;
  DevBuf w2t;   // fc2 weights transposed to [out_dim][hidden] (k contiguous)
  DevBuf part;  // split-K partials
  DevBuf conv_part;  // split-K partials of conv layers wider than the resident weight slice
  DevBuf c1acc; // calibrated conv1 accumulator row of an all-constant window (fused front)
  DevBuf calib_out;
};

namespace {

// Reference column-major W[o + k*N] -> K-major [npad][kpad], split per mode.
void upload_weights(TcWeights& w, const float* src, int n, int k, int mode, int n_tile, cudaStream_t s) {
  const int elem_per_chunk = mode_chunk_elems(mode);
  w.n = n;
  w.k = k;
  w.npad = ((n + n_tile - 1) / n_tile) * n_tile;
  w.kpad = ((k + elem_per_chunk - 1) / elem_per_chunk) * elem_per_chunk;
  const size_t cnt = static_cast<size_t>(w.npad) * w.kpad;
  if (mode == kFP8) {
    // e4m3 (max 448): a per-tensor power-of-two scale keeps the largest weight
    // near the top of the range (small weights stay out of the subnormals)
    float amax = 0.0f;
    for (int o = 0; o < n; ++o)
      for (int q = 0; q < k; ++q) amax = std::max(amax, std::fabs(src[o + static_cast<size_t>(q) * n]));
    int e = 0;
    if (amax > 0.0f) e = static_cast<int>(std::floor(std::log2(448.0f / amax)));
    e = std::max(-20, std::min(20, e));
    const float sc = std::ldexp(1.0f, e);
    w.inv_scale = std::ldexp(1.0f, -e);
    std::vector<uint8_t> h(cnt, 0);
    for (int o = 0; o < n; ++o)
      for (int q = 0; q < k; ++q)
        h[static_cast<size_t>(o) * w.kpad + q] = fp8_e4m3_host(src[o + static_cast<size_t>(q) * n] * sc);
    w.hi.need(cnt);
    CUDA_OK(cudaMemcpyAsync(w.hi.p, h.data(), cnt, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaStreamSynchronize(s));
  } else if (mode == kBF16) {
    std::vector<uint16_t> h(cnt, 0);
    for (int o = 0; o < n; ++o)
      for (int q = 0; q < k; ++q) h[static_cast<size_t>(o) * w.kpad + q] = bf16_rn_host(src[o + static_cast<size_t>(q) * n]);
    w.hi.need(cnt * 2);
    CUDA_OK(cudaMemcpyAsync(w.hi.p, h.data(), cnt * 2, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaStreamSynchronize(s));
  } else {
    std::vector<float> h(cnt, 0.0f), l(cnt, 0.0f);
    for (int o = 0; o < n; ++o)
      for (int q = 0; q < k; ++q) {
        const float x = src[o + static_cast<size_t>(q) * n];
        const float hi = tf32_round_host(x);
        h[static_cast<size_t>(o) * w.kpad + q] = hi;
        l[static_cast<size_t>(o) * w.kpad + q] = tf32_round_host(x - hi);
      }
    w.hi.need(cnt * 4);
    w.lo.need(cnt * 4);
    CUDA_OK(cudaMemcpyAsync(w.hi.p, h.data(), cnt * 4, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(w.lo.p, l.data(), cnt * 4, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaStreamSynchronize(s));
  }
  const uint64_t dims[2] = {static_cast<uint64_t>(w.kpad), static_cast<uint64_t>(w.npad)};
  const uint64_t strides[1] = {static_cast<uint64_t>(w.kpad) * mode_esz(mode)};
  const uint32_t box[2] = {static_cast<uint32_t>(elem_per_chunk), static_cast<uint32_t>(n_tile)};
  w.n_tile = n_tile;
  w.map_hi = make_map_e(w.hi.p, mode_esz(mode), 2, dims, strides, box);
  w.map_lo = mode == kTF32x3 ? make_map(w.lo.p, false, 2, dims, strides, box) : w.map_hi;
}

size_t smem_bytes(int mode, int n, int chunks, int stages, bool a_tmem = false, bool tma_multi = false,
                  int stg_bufs = 2, bool stream_w = false) {
  const size_t ns = static_cast<size_t>(stages > 0 ? stages : kStages);
  const size_t planes = mode == kTF32x3 ? 2 : 1;
  // resident slice, or (stream_w) one weight chunk per ring stage
  const size_t w = stream_w ? ns * n * 128 * planes : static_cast<size_t>(chunks) * n * 128 * planes;
  const size_t a = ns * kAChunk * (mode == kTF32x3 && !a_tmem ? 2 : 1);
  return w + a + (tma_multi ? static_cast<size_t>(stg_bufs) * kAChunk : 0) + 1024;
}

int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return g_num_sms;
}

// Split-K conv layer: out = ReLU(sum over q ascending of part[q] + bias) in a
// fixed order (batch-independent), written f32 or bf16 like the unsplit
// epilogue.  Four consecutive elements per thread.
__global__ void conv_splitk_reduce_kernel(const float* part, int nsplit, uint64_t plane, const float* bias,
                                          int cout, void* out, int out_bf16) {
  const uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i >= plane) return;
  float4 acc = *reinterpret_cast<const float4*>(part + i);
  for (int q = 1; q < nsplit; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(part + q * plane + i);
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  const int col = static_cast<int>(i % cout);
  float r[4] = {acc.x + bias[col], acc.y + bias[col + 1], acc.z + bias[col + 2], acc.w + bias[col + 3]};
  for (int j = 0; j < 4; ++j) r[j] = fmaxf(r[j], 0.0f);
  if (out_bf16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(r[0], r[1]), b = __floats2bfloat162_rn(r[2], r[3]);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&a);
    pk.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(out) + i) = pk;
  } else {
    *reinterpret_cast<float4*>(static_cast<float*>(out) + i) = make_float4(r[0], r[1], r[2], r[3]);
  }
}

void launch_mode(int mode, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& blo,
                 const CUtensorMap& out, const TcGemmParams& p, int ny, int nz, cudaStream_t s) {
  num_sms();
  const int groups = ny * nz;
  int gx = std::max(1, std::min(p.m_tiles, std::max(1, g_num_sms / groups)));
  if (p.gx_max > 0) gx = std::min(gx, p.gx_max);
  const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(ny), static_cast<unsigned>(nz));
  const size_t sm =
      smem_bytes(mode, p.n, p.chunks, p.stages, p.a_tmem != 0, p.tma_multi != 0, p.stg_bufs, p.stream_w != 0);
  if (mode == kFP8)
    launch_pdl_tag("layer_bf16", tc_layer_kernel<kFP8>, grid, dim3(kLayerThreads), sm, s, a, b, blo, out, p);
  else if (mode == kBF16)
    launch_pdl_tag("layer_bf16", tc_layer_kernel<kBF16>, grid, dim3(kLayerThreads), sm, s, a, b, blo, out, p);
  else if (mode == kTF32)
    launch_pdl_tag("layer", tc_layer_kernel<kTF32>, grid, dim3(kLayerThreads), sm, s, a, b, blo, out, p);
  else if (p.a_tmem)
    launch_pdl_tag("layer", tc_layer_kernel<kTF32x3, true>, grid, dim3(kLayerThreads), sm, s, a, b, blo, out, p);
  else
    launch_pdl_tag("layer", tc_layer_kernel<kTF32x3>, grid, dim3(kLayerThreads), sm, s, a, b, blo, out, p);
}

}  // namespace

TcModel* tc_model_create(const DevModel& m, const float* host_params, int precision, cudaStream_t s) {
  const ilsim_cnn_config& c = m.cfg;
  const int mode = mode_of(precision);
  if (c.n_conv == 0) throw ApiError("tensor-core path: the FC-only predictor runs with precision fp32");
  // constraints of this kernel family (the FP32 SIMT path has none)
  int cin = c.input_channels;
  for (int l = 0; l < c.n_conv; ++l) {
    // any input width: layers wider than kMaxChunks K chunks run split-K (tc_forward)
    if (c.conv[l] % 16 != 0 || (c.conv[l] > 128 && c.conv[l] % 128 != 0))
      throw ApiError("tensor-core path: conv channels must be multiples of 16 (and of 128 above 128)");
    cin = c.conv[l];
  }
  if (128 % (c.sequence_length / 2) != 0) throw ApiError("tensor-core path: sequence_length/2 must divide 128");
  if (c.fc_hidden % 16 != 0) throw ApiError("tensor-core path: fc_hidden must be a multiple of 16");
  CUDA_OK(cudaFuncSetAttribute(tc_layer_kernel<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  CUDA_OK(cudaFuncSetAttribute(tc_layer_kernel<kFP8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  CUDA_OK(cudaFuncSetAttribute(tc_layer_kernel<kTF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  CUDA_OK(cudaFuncSetAttribute(tc_layer_kernel<kTF32x3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  CUDA_OK(cudaFuncSetAttribute(tc_layer_kernel<kTF32x3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               226 * 1024));
  CUDA_OK(cudaFuncSetAttribute(fc_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  conv_chain_set_attributes();
  round_front_set_attributes();
  if (std::getenv("SIMNET_CHAIN_TRACE") && !chain_trace_ptr())  // diagnostics buffer, allocated outside capture
    CUDA_OK(cudaMalloc(&chain_trace_ptr(), 2 * kChainTraceWords * sizeof(long long)));
  auto* t = new TcModel();
  t->mode = mode;
  t->chain = c.n_conv == 3 && c.conv[0] == 64 && c.conv[1] == 64 && c.conv[2] == 64 && c.input_channels == 50 &&
             c.sequence_length == 128 && std::getenv("SIMNET_NO_CHAIN") == nullptr;
  try {
    cin = c.input_channels;
    for (int l = 0; l < c.n_conv; ++l) t->conv.emplace_back();
    for (int l = 0; l < c.n_conv; ++l) {
      const size_t taps = static_cast<size_t>(c.conv[l]) * 2 * cin;
      std::vector<float> w(host_params + m.L.w[l], host_params + m.L.w[l] + taps);
      // Residual blocks (c3-rb, cnn.cpp:104-107): out = W in + P in + b.  Both
      // taps read the same window, so the tensor-core path folds the shortcut
      // into the weights once (W + P in fp32); the SIMT fp32 path keeps the
      // reference's two products.
      if (c.residual)
        for (size_t i = 0; i < taps; ++i) w[i] += host_params[m.L.p[l] + i];
      upload_weights(t->conv[l], w.data(), c.conv[l], 2 * cin, mode, std::min(c.conv[l], 128), s);
      cin = c.conv[l];
    }
    // FC1 N tile: 128 hidden units for the f32 modes (one M tile per CTA at
    // K = 1024: 8 M x 2 N x 8 split planes = 128 CTAs), 64 for bf16 (4 planes),
    // else the whole (small) layer
    const int fc_tile =
        (c.fc_hidden % 128 == 0 && mode_esz(mode) == 4) ? 128 : (c.fc_hidden >= 64 ? 64 : c.fc_hidden);
    if (c.fc_hidden % fc_tile != 0) throw ApiError("tensor-core path: fc_hidden must be a multiple of 64 (or <= 64)");
    upload_weights(t->fc1, host_params + m.L.fc1_w, c.fc_hidden, m.L.flat, mode, fc_tile, s);
    // fc2 (reference column-major [od x hidden]) -> [od][hidden]
    const int od = m.L.out_dim;
    std::vector<float> w2t(static_cast<size_t>(od) * c.fc_hidden);
    for (int o = 0; o < od; ++o)
      for (int k = 0; k < c.fc_hidden; ++k)
        w2t[static_cast<size_t>(o) * c.fc_hidden + k] = host_params[m.L.fc2_w + o + static_cast<size_t>(k) * od];
    t->w2t.need(w2t.size() * 4);
    CUDA_OK(cudaMemcpyAsync(t->w2t.p, w2t.data(), w2t.size() * 4, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaStreamSynchronize(s));
  } catch (...) {
    delete t;
    throw;
  }
  return t;
}

void tc_model_destroy(TcModel* t) { delete t; }

// 128-B K chunks per FC1 split-K plane (C3 flat dim: 8 planes for the f32
// modes, 4 for bf16).  8 chunks per plane (one M tile per CTA, but only a
// 2-stage A ring fits next to the 128 KB 3xTF32 W slice) measured slower:
// the A loads are TMA-latency-bound and need the 4-stage ring.
int fc1_cps(int mode) {
  return mode == kFP8 ? 2 : kMaxChunks;  // fp8: flat is 8 chunks -> 4 planes of 2
}

// Split-K conv layers (K wider than kMaxChunks chunks): the largest layer's
// partial planes per sample (olen x cout x nsplit floats), 0 if none splits.
uint64_t conv_split_floats_per_sample(const ilsim_cnn_config& c, int esz) {
  uint64_t best = 0;
  int cin = c.input_channels, len = c.sequence_length;
  for (int l = 0; l < c.n_conv; ++l) {
    const int olen = len / 2, k = 2 * cin;
    const int nsplit = ((k * esz + 127) / 128 + kMaxChunks - 1) / kMaxChunks;
    if (nsplit > 1) best = std::max<uint64_t>(best, static_cast<uint64_t>(olen) * c.conv[l] * nsplit);
    cin = c.conv[l];
    len = olen;
  }
  return best;
}

// Allocations the forward needs, done before any graph capture.
void tc_prepare(const DevModel& m, uint64_t samples) {
  TcModel& t = *m.tc;
  const int esz = mode_esz(t.mode);
  const int total_chunks = (m.L.flat * esz + 127) / 128;
  const int nsplit = (total_chunks + fc1_cps(t.mode) - 1) / fc1_cps(t.mode);
  t.part.need(samples * static_cast<uint64_t>(m.cfg.fc_hidden) * nsplit * sizeof(float));
  if (!t.chain) {
    const uint64_t per = conv_split_floats_per_sample(m.cfg, esz);
    if (per) t.conv_part.need(samples * per * sizeof(float));
  }
}

bool tc_split_input(const TcModel* t) { return t->chain && t->mode == kTF32x3; }

uint32_t tc_act_bytes(const TcModel* t) { return static_cast<uint32_t>(mode_esz(t->mode)); }

// FC1 (split-K tcgen05 partials) and the FC tail (FC2 + fused K3) on the
// flat conv output `in`.
uint64_t tc_fc(const DevModel& m, const void* in, uint64_t samples, const ForwardBuffers& fb, cudaStream_t s,
               const DecodeParams* fuse, bool with_tail) {
  if (!m.tc) throw ApiError("internal: tensor-core model missing");
  TcModel& t = *m.tc;
  const ilsim_cnn_config& c = m.cfg;
  const int mode = t.mode;
  const int esz = mode_esz(mode);
  const int chunk_elems = mode_chunk_elems(mode);
  const float* P = m.params.as<float>();
  uint64_t launches = 0;
  // FC1 split-K partials
  const int flat = m.L.flat;
  const int total_chunks = (flat * esz + 127) / 128;
  const int per = fc1_cps(mode);
  const int nsplit = (total_chunks + per - 1) / per;
  const int fc_tile = t.fc1.n_tile;
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(flat), samples};
    const uint64_t strides[1] = {static_cast<uint64_t>(flat) * esz};
    const uint32_t box[2] = {static_cast<uint32_t>(chunk_elems), kBM};
    const CUtensorMap amap = make_map_e(in, esz, 2, dims, strides, box);
    const uint64_t plane = samples * static_cast<uint64_t>(c.fc_hidden);
    // this slice's own [nsplit][samples][hidden] block (slices run concurrently)
    const uint64_t base = fb.part_off * nsplit * static_cast<uint64_t>(c.fc_hidden);
    if (t.part.bytes < (base + plane * nsplit) * sizeof(float)) throw ApiError("internal: split-K buffer not prepared");
    float* part = t.part.as<float>() + base;
    TcGemmParams p{};
    p.m = static_cast<int>(samples);
    p.m_tiles = static_cast<int>((samples + kBM - 1) / kBM);
    p.n = fc_tile;
    p.chunks = per;
    p.ksteps_last = 4;
    // A ring depth that fits next to the resident W slice (226 KB dynamic smem)
    // 3xTF32: the split warps write A hi / lo into tensor memory and the MMAs
    // read only W from shared memory. With A in shared memory an N = 128 MMA
    // reads 8 KB per 64 cycles, all of the shared-memory bandwidth, and the
    // split's stores compete with it. (With single-thread MMA issue A from
    // shared memory was faster for CTAs with one M tile; with the warp-issued
    // MMAs A in TMEM is faster there too: c2 27.75 -> 27.40 us per round,
    // profiles/r02zo_fc1_tmem_a_c2.txt.)  SIMNET_FC1_SS: A from shared memory (A/B)
    const int groups = (t.fc1.npad / fc_tile) * nsplit;
    static const int fc1_gx = std::getenv("SIMNET_FC1_GX") ? std::atoi(std::getenv("SIMNET_FC1_GX")) : 0;
    p.gx_max = fc1_gx;
    int gx = std::max(1, std::min(p.m_tiles, std::max(1, num_sms() / groups)));
    if (p.gx_max > 0) gx = std::min(gx, p.gx_max);
    p.a_tmem = mode == kTF32x3 && p.n <= 128 && !std::getenv("SIMNET_FC1_SS");
    // CTAs that loop over M tiles TMA-store their partial tiles through two
    // staging buffers when those fit next to a full A ring (SIMNET_FC1_MULTI_DIRECT: row stores, A/B)
    const bool multi_direct = std::getenv("SIMNET_FC1_MULTI_DIRECT") != nullptr;
    p.tma_multi = p.m_tiles > gx && fc_tile % 32 == 0 && !multi_direct &&
                  smem_bytes(mode, p.n, p.chunks, kStages, p.a_tmem != 0, true) <= 226 * 1024;
    p.stg_bufs = 2;
    p.stages = kStages;
    // SIMNET_FC1_STAGES=N (A/B): an A ring N deep for CTAs looping over M tiles,
    // with one staging buffer if two do not fit
    if (const char* e = std::getenv("SIMNET_FC1_STAGES"); e && p.m_tiles > gx)
      p.stages = std::max(2, std::min(kMaxStages, std::atoi(e)));
    if (p.tma_multi && smem_bytes(mode, p.n, p.chunks, p.stages, p.a_tmem != 0, true, 2) > 226 * 1024)
      p.stg_bufs = 1;
    while (p.stages > 2 &&
           smem_bytes(mode, p.n, p.chunks, p.stages, p.a_tmem != 0, p.tma_multi != 0, p.stg_bufs) > 226 * 1024)
      --p.stages;
    p.bias = nullptr;
    p.relu = 0;
    p.out = part;
    p.ldo = c.fc_hidden;
    p.out_bf16 = 0;
    p.out_split_stride = plane;
    p.out_scale = t.fc1.inv_scale;
    p.trace = chain_trace_active();
    p.diag_skip_w = std::getenv("SIMNET_DIAG_FC1_SKIP_W") != nullptr;
    p.diag_a_early = std::getenv("SIMNET_DIAG_FC1_A_EARLY") != nullptr;
    // a last plane with fewer chunks reads TMA zero fill past the flat dim (exact zeros)
    if (nsplit > kMaxSplit) throw ApiError("tensor-core path: flat dim too large for the FC tail");
    // partial planes as a 3-D tensor [nsplit][samples][hidden]: the TMA store
    // clips rows past `samples` within each plane
    const uint64_t odims[3] = {static_cast<uint64_t>(c.fc_hidden), samples, static_cast<uint64_t>(nsplit)};
    const uint64_t ostr[2] = {static_cast<uint64_t>(c.fc_hidden) * 4, plane * 4};
    const uint32_t obox[3] = {32, 32, 1};
    const CUtensorMap omap = make_map(part, false, 3, odims, ostr, obox);
    const size_t ring = static_cast<size_t>(p.stages) * kAChunk * (mode == kTF32x3 && !p.a_tmem ? 2 : 1);
    // each solo half must be whole 32-column groups
    p.tma_out = fc_tile % 64 == 0 && ring >= static_cast<size_t>(fc_tile / 32) * kAChunk &&
                !std::getenv("SIMNET_FC1_DIRECT_STORE");
    launch_mode(mode, amap, t.fc1.map_hi, t.fc1.map_lo, omap, p, t.fc1.npad / fc_tile, nsplit, s);
    ++launches;
    if (!with_tail) return launches;  // the fused round front reduces the partials next round
    TailParams tp{};
    tp.fc = tc_fc_decode_args(m, samples, fb);
    tp.y = fb.y;
    tp.samples = static_cast<int>(samples);
    if (fuse) tp.dec = *fuse;
    const size_t tail_smem = (static_cast<size_t>(tp.fc.od + kTailWarps) * tp.fc.hidden + kTailWarps * kMaxOut) * 4;
    launch_pdl(fc_tail_kernel, dim3(static_cast<unsigned>((samples + kTailWarps - 1) / kTailWarps)),
               dim3(kTailThreads), tail_smem, s, tp);
    ++launches;
  }
  return launches;
}

bool tc_fused_front(const TcModel* t) { return t != nullptr && t->chain; }

// Calibration: one fused-front item with no sub-traces (all-zero input)
// measures the conv1 accumulator row of an all-constant window with the very
// MMA sequence the rounds use, so skipping that tile later is bit-exact.
void tc_calibrate(const DevModel& m, cudaStream_t s) {
  TcModel& t = *m.tc;
  if (!t.chain) return;
  FrontParams fp{};
  fp.first = 0;
  fp.last = 8;
  fp.max_context = m.cfg.max_context;
  fp.calibrate = 1;
  fp.c1acc_out = static_cast<float*>(t.c1acc.need(64 * sizeof(float)));
  ForwardBuffers fb{};
  fb.act[2] = static_cast<float*>(t.calib_out.need(8 * 1024 * sizeof(float)));
  tc_front(m, fp, fb, s);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaStreamSynchronize(s));
}

FcDecodeArgs tc_fc_decode_args(const DevModel& m, uint64_t samples, const ForwardBuffers& fb) {
  const TcModel& t = *m.tc;
  const ilsim_cnn_config& c = m.cfg;
  const int esz = mode_esz(t.mode);
  const int total_chunks = (m.L.flat * esz + 127) / 128;
  const int nsplit = (total_chunks + fc1_cps(t.mode) - 1) / fc1_cps(t.mode);
  if (m.L.out_dim > 64 || c.fc_hidden % 4 != 0) throw ApiError("tensor-core path: FC tail supports fc_hidden multiple of 4 and <= 64 outputs");
  if (c.fc_hidden > 256) throw ApiError("fused round front: fc_hidden must be <= 256");
  FcDecodeArgs a{};
  a.nsplit = nsplit;
  a.split_stride = samples * static_cast<uint64_t>(c.fc_hidden);
  a.part = t.part.as<float>() + fb.part_off * nsplit * static_cast<uint64_t>(c.fc_hidden);
  a.hidden = c.fc_hidden;
  a.b1 = m.params.as<float>() + m.L.fc1_b;
  a.w2t = t.w2t.as<float>();
  a.b2 = m.params.as<float>() + m.L.fc2_b;
  a.od = m.L.out_dim;
  a.class_fetch = c.class_fetch;
  a.class_exec = c.class_exec;
  a.class_store = c.class_store;
  return a;
}

// Fused round front (K1 apply + gather + conv chain) for the chunk of
// sub-traces [fp.first, fp.last); writes the flat conv2 output to fb.act[2].
uint64_t tc_front(const DevModel& m, FrontParams fp, const ForwardBuffers& fb, cudaStream_t s) {
  TcModel& t = *m.tc;
  if (!t.chain) throw ApiError("internal: fused round front needs the C3 conv chain");
  const float* P = m.params.as<float>();
  fp.b0 = P + m.L.b[0];
  fp.b1 = P + m.L.b[1];
  fp.b2 = P + m.L.b[2];
  fp.out = fb.act[2];
  CUtensorMap w[8] = {t.conv[0].map_hi, t.conv[0].map_lo, t.conv[1].map_hi, t.conv[1].map_lo,
                      t.conv[2].map_hi, t.conv[2].map_lo, t.conv[0].map_hi, t.conv[0].map_hi};
  if (fp.stat && fp.stat_rows > 0) {  // tile-0 static rows, staged by the front's producer
    const uint64_t dims[2] = {static_cast<uint64_t>(kStatStride), fp.stat_rows};
    const uint64_t strides[1] = {static_cast<uint64_t>(kStatStride) * 4};
    const uint32_t box[2] = {44, 32};
    w[7] = make_map_plain(fp.stat, 2, dims, strides, box);
  }
  const uint64_t samples = fp.last - fp.first;
  fp.out_tma = 0;
  for (int l = 0; l < 3; ++l) fp.wscale[l] = t.conv[l].inv_scale;
  if (mode_esz(t.mode) == 4 && samples > 0 && !std::getenv("SIMNET_FLAT_DIRECT_STORE")) {
    // flat as [samples * 16 rows][64 f32]: the front TMA-stores 32 x 32 boxes
    const uint64_t dims[2] = {64, samples * 16};
    const uint64_t strides[1] = {64 * 4};
    const uint32_t box[2] = {32, 32};
    w[6] = make_map(fb.act[2], false, 2, dims, strides, box);
    fp.out_tma = 1;
  }
  fp.trace = chain_trace_active();  // SIMNET_CHAIN_TRACE: event clocks of the last launch (null: off)
  if (!fp.calibrate) fp.c1acc = t.c1acc.as<float>();
  launch_round_front(t.mode, w, fp, num_sms(), s);
  return 1;
}

uint64_t tc_forward(const DevModel& m, int precision, const void* x, uint32_t x_stride, uint64_t samples,
                    const ForwardBuffers& fb, cudaStream_t s, const DecodeParams* fuse, uint64_t x_lo_off) {
  (void)precision;
  TcModel& t = *m.tc;
  const ilsim_cnn_config& c = m.cfg;
  const int mode = t.mode;
  if (mode == kFP8) throw ApiError("fp8 precision runs only the fused simulate path (no unfused forward / predict)");
  const bool bf = mode == kBF16;
  const int esz = bf ? 2 : 4;
  const int chunk_elems = bf ? 64 : 32;
  const float* P = m.params.as<float>();
  uint64_t launches = 0;

  int len = c.sequence_length;
  int cin = c.input_channels;
  const void* in = x;
  if (t.chain) {  // conv0 -> conv1 -> conv2 fused, activations stay on chip
    const uint64_t row_elems = bf ? 104 : 100;
    const uint64_t rows = x_stride / row_elems;
    const uint64_t dims[3] = {100, rows, samples};
    const uint64_t strides[2] = {row_elems * esz, static_cast<uint64_t>(x_stride) * esz};
    const uint32_t box[3] = {static_cast<uint32_t>(chunk_elems), 64, 2};
    const CUtensorMap xmap = make_map(x, bf, 3, dims, strides, box);
    if (mode == kTF32x3 && x_lo_off == 0) throw ApiError("internal: 3xTF32 chain needs split input planes");
    const CUtensorMap xlo = mode == kTF32x3
                                ? make_map(static_cast<const float*>(x) + x_lo_off, false, 3, dims, strides, box)
                                : xmap;
    const CUtensorMap w[6] = {t.conv[0].map_hi, t.conv[0].map_lo, t.conv[1].map_hi,
                              t.conv[1].map_lo, t.conv[2].map_hi, t.conv[2].map_lo};
    ChainParams cp{static_cast<int>(samples), P + m.L.b[0], P + m.L.b[1], P + m.L.b[2], fb.act[2], nullptr};
    cp.trace = chain_trace_active();  // SIMNET_CHAIN_TRACE diagnostics (null: off)
    launch_conv_chain(mode, xmap, xlo, w, cp, num_sms(), s);
    ++launches;
    in = fb.act[2];
    len = 0;
  }
  for (int l = 0; l < c.n_conv && !t.chain; ++l) {
    const int olen = len / 2, cout = c.conv[l], k = 2 * cin;
    const uint64_t m_rows = samples * olen;
    CUtensorMap amap;
    TcGemmParams p{};
    if (l == 0) {
      // gathered input: [samples][rows][row_elems]; row_elems = 100 (f32) / 104 (bf16)
      const uint64_t row_elems = bf ? 104 : 100;
      const uint64_t rows = x_stride / (bf ? 104 : 100);
      const uint64_t dims[3] = {static_cast<uint64_t>(k), rows, samples};
      const uint64_t strides[2] = {row_elems * esz, static_cast<uint64_t>(x_stride) * esz};
      const uint32_t box[3] = {static_cast<uint32_t>(chunk_elems), static_cast<uint32_t>(olen),
                               static_cast<uint32_t>(kBM / olen)};
      amap = make_map(in, bf, 3, dims, strides, box);
      p.a3d = 1;
        p.a_samples_box = kBM / olen;
    } else {
      const uint64_t dims[2] = {static_cast<uint64_t>(k), m_rows};
      const uint64_t strides[1] = {static_cast<uint64_t>(k) * esz};
      const uint32_t box[2] = {static_cast<uint32_t>(chunk_elems), kBM};
      amap = make_map(in, bf, 2, dims, strides, box);
    }
    const int bn = std::min(cout, 128);
    p.m = static_cast<int>(m_rows);
    p.m_tiles = static_cast<int>((m_rows + kBM - 1) / kBM);
    p.n = bn;
    // K wider than the resident weight slice (kMaxChunks 128-B chunks): split-K
    // over grid z, f32 partial planes, then a fixed-order reduce + bias + ReLU.
    // K past the tensor (the last split's tail) is TMA zero fill: exact zeros.
    const int total_chunks = (k * esz + 127) / 128;
    int nsplit = (total_chunks + kMaxChunks - 1) / kMaxChunks;
    // Layers with tens of thousands of rows (paper-scale models at K >= ~1k
    // sub-traces): stream the weight chunks through the ring with A instead of
    // splitting K -- one CTA per output tile accumulates all of K in TMEM, so
    // no partial planes go through HBM and no reduce kernel runs
    // (SIMNET_NO_STREAM_W: split-K, A/B)
    const bool stream = nsplit > 1 && p.m_tiles >= 64 && std::getenv("SIMNET_NO_STREAM_W") == nullptr;
    if (stream) {
      nsplit = 1;
      p.stream_w = 1;
      p.chunks = total_chunks;
      p.ksteps_last = ((k * esz + 31) / 32) - 4 * (p.chunks - 1);
    } else {
      p.chunks = nsplit > 1 ? kMaxChunks : total_chunks;
      p.ksteps_last = nsplit > 1 ? 4 : ((k * esz + 31) / 32) - 4 * (p.chunks - 1);
    }
    p.stages = kStages;
    // 3xTF32: A hi / lo split into tensor memory, the MMAs read only W from
    // shared memory (as FC1; SIMNET_LAYER_SS: A from shared memory, A/B)
    p.a_tmem = mode == kTF32x3 && p.n <= 128 && !std::getenv("SIMNET_LAYER_SS");
    while (p.stages > 2 &&
           smem_bytes(mode, p.n, p.chunks, p.stages, p.a_tmem != 0, false, 2, p.stream_w != 0) > 226 * 1024)
      --p.stages;
    p.ldo = cout;
    const uint64_t plane = m_rows * static_cast<uint64_t>(cout);
    if (nsplit == 1) {
      p.bias = P + m.L.b[l];
      p.relu = 1;
      p.out = fb.act[l];
      p.out_bf16 = bf;
    } else {
      // this slice's own block (slices of one round run concurrently), prepared by tc_prepare
      const uint64_t per = conv_split_floats_per_sample(c, esz);
      if (t.conv_part.bytes < (fb.part_off + samples) * per * sizeof(float))
        throw ApiError("internal: conv split-K buffer not prepared");
      float* part = t.conv_part.as<float>() + fb.part_off * per;
      p.bias = nullptr;
      p.relu = 0;
      p.out = part;
      p.out_bf16 = 0;
      p.out_split_stride = plane;
    }
    launch_mode(mode, amap, t.conv[l].map_hi, t.conv[l].map_lo, amap, p, cout / bn, nsplit, s);  // no TMA store
    ++launches;
    if (nsplit > 1) {
      const float* part_conv = static_cast<const float*>(p.out);
      const uint64_t threads = plane / 4;
      conv_splitk_reduce_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
          part_conv, nsplit, plane, P + m.L.b[l], cout, fb.act[l], bf);
      CUDA_OK(cudaGetLastError());
      ++launches;
    }
    in = fb.act[l];
    cin = cout;
    len = olen;
  }
  return launches + tc_fc(m, in, samples, fb, s, fuse, true);
}

}  // namespace simnet
