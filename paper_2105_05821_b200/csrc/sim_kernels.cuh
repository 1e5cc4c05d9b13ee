// Launch interfaces of the simulation kernels (K1 context-queue, K3 decode,
// pack).  Parameter blocks are passed by value so launches capture cleanly
// into CUDA graphs.
#pragma once
#include "common.cuh"

namespace simnet {

constexpr int kCtxThreads = 128;  // K1 block: one sub-trace per block (warp 0 applies, all gather)
constexpr int kMaxCols = 128;   // max_context + 1 supported by the gather (C3: 111)

struct CtxParams {
  SubState* state;
  RingEntry* proc;
  RingEntry* wq;
  uint32_t pmask, wmask;     // ring capacities - 1 (powers of two)
  uint64_t first, last;      // sub-trace range of this launch (chunk)
  const float* stat;         // [n][kStatStride] normalised static slots
  const uint64_t* pc;
  const uint64_t* addr;
  const uint8_t* iflags;
  const NormConsts* nc;
  void* x;                   // [last-first][x_stride] gathered inputs (f32 or bf16)
  uint32_t x_stride;         // elements per sample in x
  uint32_t x_floats;         // logical floats per sample (100 per conv0 row, multiple of 4)
  int32_t x_bf16;            // 1: rows of 104 bf16 (100 + zero pad, TMA-aligned)
  int32_t x_full;            // 1: rewrite whole rows (x rows shared between chunks)
  int32_t x_split;           // 1: 3xTF32 planes: x = tf32 hi, x + x_lo_off = lo (x - hi)
  uint64_t x_lo_off;         // elements from the hi plane to the lo plane
  int32_t max_context;
  uint32_t bw, line, page;
  int32_t per_cycle;
  int32_t gather;
};

struct DecodeParams {
  SubState* state;
  uint64_t first, last;
  const float* y;            // [last-first][y_stride] head outputs (null in oracle mode)
  uint32_t y_stride;
  const uint32_t* truth;     // oracle mode: [n][3]
  const uint8_t* iflags;
  const NormConsts* nc;
  uint32_t* pred_fetch;      // owned predicted fetch series (may be null)
  int32_t class_fetch, class_exec, class_store;
  int32_t per_cycle;
};

struct PackParams {
  uint64_t n;
  const uint8_t* op;
  const uint16_t* src;
  const uint16_t* dst;
  const uint16_t* hist;
  const NormConsts* nc;
  float* stat;               // may be null (oracle mode)
  uint8_t* iflags;
  // segmented mode (seg_len > 0): instructions seg_first + s * seg_stride + o,
  // s < n / seg_len, o < seg_len (one window of equal-length sub-traces)
  uint64_t seg_first, seg_stride, seg_len;
};

void launch_ctx(const CtxParams& p, cudaStream_t stream);
void launch_decode(const DecodeParams& p, cudaStream_t stream);
void launch_decode_only(const float* y, int y_stride, uint64_t n, const uint8_t* is_store,
                        const NormConsts* nc, int cf, int ce, int cs, uint32_t* out,
                        cudaStream_t stream);
// Same decode, the fused round's warp-cooperative form (test hook).
void launch_decode_warp(const float* y, int y_stride, uint64_t n, const uint8_t* is_store,
                        const NormConsts* nc, int cf, int ce, int cs, uint32_t* out,
                        cudaStream_t stream);
void launch_pack(const PackParams& p, cudaStream_t stream);

// SNT1 records (108 B, trace.cpp:49-83) -> device structure-of-arrays.
struct UnpackParams {
  const uint8_t* rec;  // n records
  uint64_t n;
  uint64_t* pc;
  uint64_t* addr;
  uint8_t* op;         // [n][13]
  uint16_t* src;       // [n][8]
  uint16_t* dst;       // [n][6]
  uint16_t* hist;      // [n][14]
  uint32_t* truth;     // [n][3] or null
};
void launch_unpack_records(const UnpackParams& p, cudaStream_t stream);
// Caller inputs [n][width] f32 -> gathered-input layout (ilsim_gpu_predict).
void launch_pack_inputs(const float* in, uint64_t n, uint32_t width, void* x, uint32_t x_stride, int x_bf16,
                        uint64_t x_lo_off, cudaStream_t stream);

}  // namespace simnet
