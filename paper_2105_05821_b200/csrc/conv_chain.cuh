// Fused conv0 -> conv1 -> conv2 kernel (tensor cores) for the C3 preset.
#pragma once
#include <cuda.h>
#include <cstdint>

#include "host_util.cuh"

namespace simnet {

struct ChainParams {
  int samples;
  const float* b0;
  const float* b1;
  const float* b2;
  void* out;  // flat [samples][1024] (f32, or bf16 for the bf16 path)
  long long* trace;  // optional: per-CTA event clocks (diagnostics, SIMNET_CHAIN_TRACE)
};

// w: {W0 hi, W0 lo, W1 hi, W1 lo, W2 hi, W2 lo} tensor maps (box 1 chunk x 64 rows)
// x / xlo: gathered input planes (xlo: 3xTF32 lo plane, ignored otherwise)
void launch_conv_chain(int mode, const CUtensorMap& x, const CUtensorMap& xlo, const CUtensorMap* w,
                       const ChainParams& p, int num_sms, cudaStream_t s);
void conv_chain_set_attributes();
size_t chain_smem_bytes();
inline long long*& chain_trace_ptr() {
  static long long* p = nullptr;
  return p;
}
// Diagnostics: whether the launch being recorded writes the trace buffer (the
// round loop traces one mid-graph round instead of the final one).
inline bool& chain_trace_on() {
  static bool on = true;
  return on;
}
// Two consecutive rounds are traced into slots 0 and 1 (kChainTraceWords each).
constexpr int kChainTraceFrontX = 148 * 32 + 256 * 32;  // front extras: 16 words per CTA
constexpr int kChainTraceWords = kChainTraceFrontX + 148 * 16;
inline int& chain_trace_slot() {
  static int slot = 0;
  return slot;
}
inline long long* chain_trace_active() {
  return chain_trace_on() && chain_trace_ptr() ? chain_trace_ptr() + chain_trace_slot() * kChainTraceWords : nullptr;
}

}  // namespace simnet
