// K3 logic shared by the standalone decode kernel and the fused inference
// tail: hybrid decode (cnn.cpp:388-417) and the fetch-clock advance
// (advance_cycles(F, bw*F), simcore.cpp:117-123, 147-149).
#pragma once
#include "common.cuh"

namespace simnet {

__device__ __forceinline__ uint32_t decode_head(const float* y, int base, int n, float r, double mu,
                                                double sigma) {
  int best = 0;
  float bv = y[base];
  for (int i = 1; i < n; ++i) {
    const float v = y[base + i];
    if (v > bv) {  // strict: first maximum wins, NaN never wins (cnn.cpp:388-393)
      bv = v;
      best = i;
    }
  }
  if (best < n - 1) return static_cast<uint32_t>(best);
  // overflow class: de-normalise out of log1p space (cnn.cpp:399-401); the
  // reference's -march=native build contracts r*sigma+mu into one fp64 FMA.
  // std::min / std::max operand order (a NaN regression passes min and max
  // turns it into 0, as in the reference; fmin/fmax would drop the NaN instead)
  const double x = fma(static_cast<double>(r), sigma, mu);
  const double z = (22.0 < x) ? 22.0 : x;        // std::min(x, 22.0)
  const double e = expm1(z);
  const double raw = (0.0 < e) ? e : 0.0;        // std::max(0.0, e)
  const long long v = llround((4.0e9 < raw) ? 4.0e9 : raw);  // std::min(raw, 4.0e9)
  return static_cast<uint32_t>(v > 0xffffffffLL ? 0xffffffffLL : v);
}

__device__ __forceinline__ void decode_triple(const float* y, const NormConsts& nc, int cf, int ce, int cs,
                                              bool is_store, uint32_t* out) {
  out[0] = decode_head(y, 3, cf, y[0], nc.label_mean[0], nc.label_sd[0]);
  const uint32_t e = decode_head(y, 3 + cf, ce, y[1], nc.label_mean[1], nc.label_sd[1]);
  out[1] = e < 1u ? 1u : e;
  out[2] = is_store ? decode_head(y, 3 + cf + ce, cs, y[2], nc.label_mean[2], nc.label_sd[2]) : 0u;
}

// Record the decoded step for instruction `pos`; K1 of the next round applies it.
__device__ __forceinline__ void apply_decoded(SubState* sp, const uint32_t* t, uint32_t* pred_fetch,
                                              int per_cycle) {
  const uint32_t pos = sp->pos;
  sp->pend_f = t[0];
  sp->pend_e = t[1];
  sp->pend_s = t[2];
  sp->has_pend = 1;
  if (!per_cycle && t[0] > 0) sp->cur += t[0];  // advance_cycles(F, ...): cur += F
  if (pos >= sp->warm) {
    sp->sum_fetch += t[0];
    if (pred_fetch) pred_fetch[sp->fetch_off + (pos - sp->warm)] = t[0];
  }
}

}  // namespace simnet
