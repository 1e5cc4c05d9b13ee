// Persistent cooperative kernel for the FC-only predictor at small K (seq_fc.cu).
#pragma once
#include "sim_kernels.cuh"

namespace simnet {

struct SeqFcParams {
  CtxParams ctx;         // K1 for the sub-traces [ctx.first, ctx.last); ctx.x: f32 rows of ctx.x_stride
  DecodeParams dec;      // K3; dec.y: [K][y_stride] head outputs
  const float* w1;       // FC1 [flat][hidden] (reference layout W[o + k * hidden])
  const float* b1;
  const float* w2;       // FC2 [hidden][od]
  const float* b2;
  int32_t flat, hidden, od;
  int32_t max_outs;      // hidden units per worker CTA (set by the launcher)
  float* h;              // [K][hidden] hidden layer (global, between the CTAs)
  float* y;              // [K][dec.y_stride] head outputs (dec.y, writable)
  uint32_t* flags;       // [0] rows published (round + 1, or ~0 = exit), [1] hidden-slice count, [2] error
  uint32_t rounds;
  long long* trace;      // diagnostics (SIMNET_SEQ_TRACE): %globaltimer at phase boundaries of one round
};

bool seq_fc_fits(int flat, int hidden, int od, int K, int ctas, int pcap);

// The C3 (3 x 64-channel conv, 50 x 128 input) at ONE sub-trace, fp32.
struct SeqC3Params {
  CtxParams ctx;         // K1 for the sub-trace [ctx.first, ctx.first + 1); ctx.x is replaced by shared memory
  DecodeParams dec;      // K3
  const float *w0, *b0, *w1c, *b1c, *w2c, *b2c;  // conv weights [2 cin][64] (reference layout) and biases
  const float *w1f, *b1f;                         // FC1 [1024][hidden]
  const float *w2f, *b2f;                         // FC2 [hidden][od]
  int32_t hidden, od;
  float* flat;           // [1024] conv2 output (global, control -> workers)
  float* h;              // [hidden] FC1 output (global, workers -> control)
  uint32_t* flags;       // [0] flat published (round + 1, or ~0 = exit), [1] hidden-slice count, [2] error
  uint32_t rounds;
  long long* trace;      // diagnostics (SIMNET_SEQ_TRACE): %globaltimer at phase boundaries of one round
};
bool seq_c3_fits(int hidden, int od, int ctas, int pcap);
void launch_seq_c3(SeqC3Params p, int ctas, cudaStream_t s);
void launch_seq_fc(SeqFcParams p, int ctas, cudaStream_t s);

}  // namespace simnet
