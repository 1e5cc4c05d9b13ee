// Warp-cooperative FC tail for one sample: h = ReLU(sum of FC1 split-K
// partials + b1), y = W2 h + b2, hybrid decode (cnn.cpp:106-125, 388-417).
// Shared by the FC tail kernel (unfused path, teacher-forced predict), the
// fused round front (decoding the previous round's prediction right before
// applying it) and the final decode/drain kernel, so every path computes the
// same bits.  Fixed, batch-independent arithmetic order:
//   lane l owns hidden units 4c..4c+3 for c = l, l + 32 (c < hidden/4);
//   h_j = ReLU((sum_q part[q][j], q ascending from 0) + b1[j]);
//   y_o = (transpose-reduction over lanes of each lane's fma chain over its
//          units: exchange stages xor 16, 8, 4, 2, 1) + b2[o].
#pragma once
#include "common.cuh"
#include "decode.cuh"
#include "tc_common.cuh"

namespace simnet {

constexpr int kFcMaxHidden = 256;
constexpr int kFcMaxSplit = 8;
constexpr int kFcMaxOut = 64;

struct FcDecodeArgs {
  const float* part;      // [nsplit][split_stride] : [samples][hidden] per split plane
  int32_t nsplit;
  uint64_t split_stride;
  int32_t hidden;         // multiple of 4, <= 256
  const float* b1;
  const float* w2t;       // [od][hidden] (global; callers stage it in shared memory)
  const float* b2;
  int32_t od;             // output_dim <= 64
  int32_t class_fetch, class_exec, class_store;
  uint32_t* pred_fetch;   // owned predicted fetch series (may be null)
  int32_t per_cycle;
};

__device__ __forceinline__ void fc_sync256() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Hybrid decode of one sample's head outputs y (decode_triple, decode.cuh),
// the three heads on lanes 0-2 in parallel; returns the triple in every lane.
// lab: label mean[3], stdev[3] (NormStats, dataset.hpp:54-65), in shared memory.
__device__ __forceinline__ void warp_decode_triple(const float* y, const double* lab, int cf, int ce, int cs,
                                                   bool is_store, uint32_t* t) {
  const int lane = threadIdx.x & 31;
  uint32_t mine = 0;
  if (lane < 3) {
    const int base = lane == 0 ? 3 : (lane == 1 ? 3 + cf : 3 + cf + ce);
    const int n = lane == 0 ? cf : (lane == 1 ? ce : cs);
    mine = decode_head(y, base, n, y[lane], lab[lane], lab[3 + lane]);
    if (lane == 1) mine = mine < 1u ? 1u : mine;  // execution >= 1
    if (lane == 2 && !is_store) mine = 0u;       // store latency only for stores
  }
  t[0] = __shfl_sync(0xffffffffu, mine, 0);
  t[1] = __shfl_sync(0xffffffffu, mine, 1);
  t[2] = __shfl_sync(0xffffffffu, mine, 2);
}

// FC tail of 8 samples by the 8 warps (256 threads, named barrier 1) of a
// CTA; warp w owns sample w.  s_local[w]: the sample's row in the partial
// planes (any valid row for an unused warp).  w2s: W2 [od][hidden] in shared
// memory; hs: 8 x hidden floats and ys: 8 x 64 floats of shared scratch (ys
// holds y on return).  Arithmetic order (fixed, batch-independent):
//   h[s][j] = ReLU((sum over q ascending of part[q][s][j]) + b1[j]);
//   lane l owns hidden units 4c..4c+3, c = l, l + 32: its partial for (s, o) is
//   an fma chain over those units in order; the 32 lane partials of the 8
//   samples are combined by a transpose reduction (xor 16, 8, 4) then a
//   butterfly (xor 2, 1); y[s][o] = that + b2[o].
// w2_bar: when non-null, W2 is still landing (bulk copy): wait on this
// mbarrier phase parity right before FC2, after the partials are reduced.
// part_smem: the CTA's 8 partial rows per plane in shared memory,
// [q][8][hidden] (landing on part_bar, phase parity part_parity); every
// thread then arrives on read_bar once its partials are consumed.
__device__ inline void cta8_fc(const FcDecodeArgs& a, uint64_t s_local, const float* w2s, float* hs, float* ys,
                               long long* trace = nullptr, uint64_t* w2_bar = nullptr, uint32_t w2_parity = 0,
                               const float* part_smem = nullptr, uint64_t* part_bar = nullptr,
                               uint64_t* read_bar = nullptr, uint32_t part_parity = 0) {
  const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
  const int hid = a.hidden, c4 = hid >> 2;
  // biases fetched with the partials (no dependent global load later): lane j
  // holds b2 of this warp's j-th output, b1 of its own hidden units
  const float b2v = (lane < 8 && warp + 8 * lane < a.od) ? __ldg(a.b2 + warp + 8 * lane) : 0.0f;
  // and lane i < od % 8 holds b2 of remainder output (od & ~7) + i
  const float b2r = lane < (a.od & 7) ? __ldg(a.b2 + (a.od & ~7) + lane) : 0.0f;
  float4 b1v[2];
#pragma unroll
  for (int u = 0; u < 2; ++u)
    b1v[u] = lane + 32 * u < c4 ? __ldg(reinterpret_cast<const float4*>(a.b1) + lane + 32 * u)
                                : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  {  // h of this warp's sample
    float4 pv[2][kFcMaxSplit];
    if (part_smem) {
      mbar_wait(part_bar, part_parity);
      const float4* ps = reinterpret_cast<const float4*>(part_smem + warp * hid);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane + 32 * u;
#pragma unroll
        for (int q = 0; q < kFcMaxSplit; ++q)
          pv[u][q] = (c < c4 && q < a.nsplit) ? ps[q * 2 * hid + c] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane + 32 * u;
#pragma unroll
        for (int q = 0; q < kFcMaxSplit; ++q)
          pv[u][q] = (c < c4 && q < a.nsplit)
                         ? __ldg(reinterpret_cast<const float4*>(a.part + q * a.split_stride + s_local * hid) + c)
                         : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = lane + 32 * u;
      if (c >= c4) continue;
      float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < kFcMaxSplit; ++q) {  // fixed order (zeros past nsplit are exact)
        acc.x += pv[u][q].x;
        acc.y += pv[u][q].y;
        acc.z += pv[u][q].z;
        acc.w += pv[u][q].w;
      }
      const float4 b = b1v[u];
      reinterpret_cast<float4*>(hs + warp * hid)[c] =
          make_float4(fmaxf(acc.x + b.x, 0.0f), fmaxf(acc.y + b.y, 0.0f), fmaxf(acc.z + b.z, 0.0f),
                      fmaxf(acc.w + b.w, 0.0f));
    }
  }
  if (part_smem) mbar_arrive(read_bar);  // partials consumed (they fed the h stores above)
  if (w2_bar) mbar_wait(w2_bar, w2_parity);
  fc_sync256();
  if (trace && threadIdx.x == 0) trace[0] = clock64();
  {  // FC2: warp w computes outputs o = w, w + 8, ... for all 8 samples; the
     // od % 8 remainder outputs are spread one sample per warp
    float4 hr[8][2];
#pragma unroll
    for (int sm = 0; sm < 8; ++sm)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane + 32 * u;
        hr[sm][u] = c < c4 ? reinterpret_cast<const float4*>(hs + sm * hid)[c] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
    auto row = [&](int o, float4 (&wv)[2]) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane + 32 * u;
        wv[u] = c < c4 ? reinterpret_cast<const float4*>(w2s + o * hid)[c] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
    };
    auto dot = [&](const float4 (&wv)[2], const float4 (&hv)[2]) {  // this lane's 8 hidden units
      float p = 0.0f;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        p = fmaf(wv[u].x, hv[u].x, p);
        p = fmaf(wv[u].y, hv[u].y, p);
        p = fmaf(wv[u].z, hv[u].z, p);
        p = fmaf(wv[u].w, hv[u].w, p);
      }
      return p;
    };
    // lane sums over xor 16, 8, 4, 2, 1 (the butterfly below pairs lanes the
    // same way, and fp addition is commutative: every output rounds identically)
    auto transpose_store = [&](float (&v)[8], int o, float b2o) {
#pragma unroll
      for (int m = 16, n = 4; m >= 4; m >>= 1, n >>= 1) {  // transpose: 8 -> 4 -> 2 -> 1 values per lane
        const bool upper = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const float keep = upper ? v[i + n] : v[i];
          const float send = upper ? v[i] : v[i + n];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
      }
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
      if ((lane & 3) == 0) {
        const int sm = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
        ys[sm * kFcMaxOut + o] = v[0] + b2o;
      }
    };
    const int full = a.od >> 3;
    for (int j = 0; j < full; ++j) {
      const int o = warp + 8 * j;
      const float b2o = __shfl_sync(0xffffffffu, b2v, j);
      float4 wv[2];
      row(o, wv);
      float v[8];
#pragma unroll
      for (int sm = 0; sm < 8; ++sm) v[sm] = dot(wv, hr[sm]);
      transpose_store(v, o, b2o);
    }
    // remainder outputs 8 * full + i: warp w takes sample w (its h re-read from smem)
    const int rem = a.od & 7;
    if (rem) {
      float4 hv[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane + 32 * u;
        hv[u] = c < c4 ? reinterpret_cast<const float4*>(hs + warp * hid)[c] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
      for (int i = 0; i < rem; ++i) {
        const int o = 8 * full + i;
        float4 wv[2];
        row(o, wv);
        float p = dot(wv, hv);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) p += __shfl_xor_sync(0xffffffffu, p, m);
        const float b2o = __shfl_sync(0xffffffffu, b2r, i);
        if (lane == 0) ys[warp * kFcMaxOut + o] = p + b2o;
      }
    }
  }
  fc_sync256();
}

// apply_decoded (decode.cuh) on a register copy of the state; lane 0 records
// the predicted fetch latency.
__device__ __forceinline__ void apply_decoded_reg(SubState& st, const uint32_t* t, uint32_t* pred_fetch,
                                                  int per_cycle) {
  const uint32_t pos = st.pos;
  st.pend_f = t[0];
  st.pend_e = t[1];
  st.pend_s = t[2];
  st.has_pend = 1;
  if (!per_cycle && t[0] > 0) st.cur += t[0];
  if (pos >= st.warm) {
    st.sum_fetch += t[0];
    if (pred_fetch && (threadIdx.x & 31) == 0) pred_fetch[st.fetch_off + (pos - st.warm)] = t[0];
  }
}

}  // namespace simnet
