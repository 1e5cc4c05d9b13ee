// K1 device body shared by ctx_kernel (sim_kernels.cu) and the persistent
// FC-predictor kernel (seq_fc.cu).
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "k1_device.cuh"
#include "sim_kernels.cuh"

namespace simnet {

// K1 for sub-trace s by a block of NT threads (the body of ctx_kernel; the
// persistent FC kernel runs it for its sub-traces in turn): warp 0 applies the
// pending step, then all NT threads build the column descriptors and write
// the gathered row (simcore.cpp:25-66, 112-159).
struct CtxSmem {
  uint32_t inst[kMaxCols];                // instruction of each column
  float dyn[kMaxCols][kSlots - kStatic];  // its 9 dynamic slots, normalised
  SubState st;                            // state after the apply step
};

template <int NT>
__device__ __forceinline__ void ctx_one(const CtxParams& p, uint64_t s, CtxSmem& sm) {
  uint32_t* s_inst = sm.inst;
  auto& s_dyn = sm.dyn;
  SubState& s_st = sm.st;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = k1::lane_id();
  if (s >= p.last) return;

  SubState* sp = p.state + s;
  const NormConsts& nc = *p.nc;
  const k1::Rings r = k1::rings_of(p.proc, p.wq, p.pmask, p.wmask, s);
  if (warp == 0) {
    SubState st = *sp;  // every lane holds a copy; lane 0 writes back
    if (st.status == kOk && st.has_pend) {
      const k1::ApplyArgs aa{p.bw, p.max_context, p.per_cycle, p.gather, p.iflags, p.nc};
      k1::apply_step(st, r, aa);
      if (lane == 0) *sp = st;
      __syncwarp();
    }
    if (lane == 0) s_st = st;
  }
  __syncthreads();
  const SubState st = s_st;
  if (!p.gather || st.status != kOk || st.pos >= st.len) return;

  // ---- gather (simcore.cpp:25-66) --------------------------------------
  const uint64_t tgt = st.begin + st.pos;
  const uint32_t nproc = st.pt - st.ph;
  const uint32_t nwq = st.wt - st.wh;
  const uint32_t ncols = min(static_cast<uint32_t>(p.max_context), nproc + nwq);
  const uint64_t tpc = p.pc[tgt];
  const uint64_t taddr = p.addr[tgt];
  const bool tmem = (p.iflags[tgt] & kFlagMem) != 0;
  // Column descriptors, 4 columns per lane in flight: ring entry, then the
  // context instruction's pc/address/flags (newest first: proc, then write
  // queue).  Loads are unconditional from clamped, always-valid addresses so
  // they issue back to back; predicates only select the results.
  for (uint32_t c = tid; c <= ncols; c += NT) {
    if (c == 0) {
      s_inst[0] = static_cast<uint32_t>(tgt);
#pragma unroll
      for (int k = kStatic; k < kSlots; ++k) s_dyn[0][k - kStatic] = nc.zero[k];
      continue;
    }
    const RingEntry e = k1::context_entry(st, r, c - 1);
    const int32_t res = static_cast<int32_t>(static_cast<uint32_t>(st.cur - e.push));
    const uint32_t f = k1::dep_flags(tpc, taddr, tmem, e, p.line, p.page);
    float* d = s_dyn[c];
    s_inst[c] = static_cast<uint32_t>(st.begin + e.idx);
    d[0] = norm_slot(res, nc.mean[kSlotResidence], nc.sd[kSlotResidence]);
    d[1] = e.nexec;
    d[2] = e.nstore;
#pragma unroll
    for (int b = 0; b < 5; ++b) d[3 + b] = ((f >> b) & 1u) ? nc.one[kSlotFlag0 + b] : nc.zero[kSlotFlag0 + b];
    d[8] = nc.zero[kSlotReserved];
  }
  __syncthreads();

  // Row write: live columns, then zeros only where the previous round of this
  // sub-trace left non-zero columns (the rest of the row is already 0).  The
  // 16 static-slot loads of an iteration are unconditional (clamped index).
  const uint32_t live = (ncols + 1) * kSlots;
  const uint32_t prev = p.x_full ? p.x_floats : st.xcols * kSlots;
  const uint32_t n4 = ((live > prev ? live : prev) + 3) / 4;
  float4* out4 = reinterpret_cast<float4*>(static_cast<float*>(p.x) + (s - p.first) * static_cast<uint64_t>(p.x_stride));
  __nv_bfloat16* outb = static_cast<__nv_bfloat16*>(p.x) + (s - p.first) * static_cast<uint64_t>(p.x_stride);
  for (uint32_t q0 = 0; q0 < n4; q0 += 4 * NT) {
    float stv[4][4], dyv[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t jf = 4 * (q0 + u * NT + tid) + t;
        const uint32_t col = jf / kSlots, slot = jf - col * kSlots;
        const uint32_t colc = jf < live ? col : 0u;
        const bool st_slot = slot < kStatic;
        stv[u][t] = __ldg(p.stat + static_cast<uint64_t>(s_inst[colc]) * kStatStride + (st_slot ? slot : 0u));
        dyv[u][t] = s_dyn[colc][st_slot ? 0u : slot - kStatic];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t q = q0 + u * NT + tid;
      float v[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t jf = 4 * q + t;
        const uint32_t slot = jf - (jf / kSlots) * kSlots;
        const float val = slot < kStatic ? stv[u][t] : dyv[u][t];
        v[t] = jf < live ? val : 0.0f;
      }
      if (q >= n4) continue;
      if (p.x_bf16) {
        const uint32_t row = (4 * q) / 100, within = 4 * q - 100 * row;
        __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&a);
        w.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(outb + row * 104 + within) = w;
      } else if (p.x_split) {  // 3xTF32: hi = tf32 round-half-away (cvt.rna), lo = v - hi (exact)
        float h[4], l[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          h[t] = __uint_as_float((__float_as_uint(v[t]) + 0x1000u) & 0xffffe000u);
          l[t] = v[t] - h[t];
        }
        out4[q] = make_float4(h[0], h[1], h[2], h[3]);
        reinterpret_cast<float4*>(reinterpret_cast<float*>(out4) + p.x_lo_off)[q] = make_float4(l[0], l[1], l[2], l[3]);
      } else {
        out4[q] = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
  }
  if (tid == 0) {
    sp->xcols = ncols + 1;
    sp->t_pc = tpc;  // the next round's push carries these into the ring entry
    sp->t_addr = taddr;
    sp->t_flags = p.iflags[tgt];
  }
}


}  // namespace simnet
