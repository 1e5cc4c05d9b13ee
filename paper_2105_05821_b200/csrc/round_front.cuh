// Fused round front: K1 (apply step + drain + context gather) and the conv
// chain of K2 in one kernel.  The gathered input never leaves the SM: it is
// written straight into the SWIZZLE_128B conv0 operand in shared memory.
#pragma once
#include <cuda.h>
#include <cstdint>

#include "common.cuh"
#include "fc_decode.cuh"
#include "host_util.cuh"

namespace simnet {

struct FrontParams {
  // K1 (same meaning as CtxParams)
  SubState* state;
  RingEntry* proc;
  RingEntry* wq;
  uint32_t pmask, wmask;
  uint64_t first, last;      // sub-trace range of this launch (chunk)
  const float* stat;         // [n][kStatStride] normalised static slots
  uint64_t stat_rows;        // n (rows of the static table on the device)
  const uint64_t* pc;
  const uint64_t* addr;
  const uint8_t* iflags;
  const NormConsts* nc;
  int32_t max_context;
  uint32_t bw, line, page;
  int32_t per_cycle;
  // conv chain
  const float* b0;
  const float* b1;
  const float* b2;
  float wscale[3];           // fp8: per-layer accumulator scale (1 / weight scale); 1 otherwise
  void* out;                 // flat [last-first][1024] (f32, or bf16 for the bf16 path)
  int32_t out_tma;           // f32 flat: staged in shared memory and TMA-stored through w[6]
  // optional: write the gathered input (exact f32 values) in the standard
  // row layout [last-first][dump_stride] (rows of 100 floats) — input capture
  float* dump;
  uint32_t dump_stride;
  // FC tail of the previous round (decoded here, right before its apply step)
  FcDecodeArgs fc;
  // conv1 accumulator row of an all-constant input window (conv0 = ReLU(b0) on
  // both taps), measured once per model by a calibration launch; lets an item
  // whose contexts fit in 64 columns skip the all-constant conv1 tile.  Null:
  // never skip.
  const float* c1acc;
  float* c1acc_out;          // calibration launch: where to write it
  int32_t calibrate;         // 1: no sub-traces, all-zero input (calibration)
  long long* trace;          // optional: per-CTA event clocks of the first item (diagnostics)
};

// w: {W0 hi, W0 lo, W1 hi, W1 lo, W2 hi, W2 lo} tensor maps (box 1 chunk x 64 rows),
//    w[6]: flat viewed as [(last-first)*16 rows][64 f32], box 32 x 32, SWIZZLE_128B (p.out_tma),
//    w[7]: the static-slot table viewed as [trace rows][48 f32], box 44 x 32, no swizzle
void launch_round_front(int mode, const CUtensorMap* w, const FrontParams& p, int num_sms, cudaStream_t s);
void round_front_set_attributes();
// After the last round: decode the outstanding predictions, apply them and
// drain (the fused-path replacement of the final K1 pass).
void launch_final_decode(const FrontParams& p, cudaStream_t s);

}  // namespace simnet
