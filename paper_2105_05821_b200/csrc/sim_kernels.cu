// K1 (context-queue), K3 (decode + clock) and the trace pack kernel.
//
// K1 replaces, per sub-trace and per round, SimCore::apply_step's retire /
// stall / push half (simcore.cpp:112-150 after the fetch advance), drain
// (simcore.cpp:152-159) and next_request (simcore.cpp:25-66).  One warp owns
// one sub-trace: ring heads are scanned 32 entries at a time with ballots
// (in-order retirement = the run of leading ready entries), store moves to
// the write queue are a ballot/popc compaction, and the gathered context is
// staged per column in shared memory and written as coalesced float4 rows.
//
// K3 replaces decode_hybrid (cnn.cpp:388-417) plus the clock half of
// apply_step (advance_cycles(F, bw*F), simcore.cpp:117-123, 147-149).
#include <cuda_bf16.h>

#include "common.cuh"
#include "decode.cuh"
#include "launch.cuh"
#include "sim_kernels.cuh"

namespace simnet {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t leading_run(uint32_t mask) {
  return mask == kFull ? 32u : static_cast<uint32_t>(__ffs(~mask) - 1);
}

struct Rings {
  RingEntry* proc;
  RingEntry* wq;
  uint32_t pmask, wmask, wcap;
};

// SimCore::retire (simcore.cpp:68-84).  Warp-uniform in/out; returns the
// number of queue transitions.  Sets *err on write-ring overflow.
__device__ uint32_t warp_retire(uint64_t cur, uint64_t budget, const Rings& r, uint32_t& ph,
                                uint32_t pt, uint32_t& wh, uint32_t& wt, uint32_t* err) {
  const uint32_t lane = lane_id();
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t events = 0;
  while (budget > 0 && ph != pt) {
    const uint32_t n = min(pt - ph, 32u);
    RingEntry e;
    bool ready = false;
    if (lane < n) {
      e = r.proc[(ph + lane) & r.pmask];
      ready = (cur - e.push) >= e.exec;
    }
    const uint32_t run = leading_run(__ballot_sync(kFull, ready));
    const uint32_t take = static_cast<uint32_t>(min(static_cast<uint64_t>(run), budget));
    const bool mv = lane < take && (e.flags & kFlagStore);
    const uint32_t sm = __ballot_sync(kFull, mv);
    const uint32_t nmv = __popc(sm);
    if (wt + nmv - wh > r.wcap) {
      *err = kErrWriteRing;
      return events;
    }
    if (mv) r.wq[(wt + __popc(sm & lt)) & r.wmask] = e;
    wt += nmv;
    ph += take;
    budget -= take;
    events += take;
    if (take < n) break;
  }
  while (wh != wt) {
    const uint32_t n = min(wt - wh, 32u);
    bool ready = false;
    if (lane < n) {
      const RingEntry& e = r.wq[(wh + lane) & r.wmask];
      ready = (cur - e.push) >= e.store;
    }
    const uint32_t run = leading_run(__ballot_sync(kFull, ready));
    wh += run;
    events += run;
    if (run < n) break;
  }
  __syncwarp();
  return events;
}

// readiness gap of a head entry (simcore.cpp:95-110 per queue)
__device__ __forceinline__ uint64_t head_gap(uint64_t cur, uint64_t push, uint32_t lat) {
  const uint64_t res = cur - push;
  return lat > res ? lat - res : 1;
}

}  // namespace

// ---------------------------------------------------------------------------
// K1: apply the pending step, drain finished sub-traces, gather the next input.
// One 128-thread block per sub-trace: warp 0 runs the (inherently serial)
// queue update with warp ballots; then all 128 threads gather, one column
// descriptor per thread and one coalesced pass over the row, so the gather is
// two dependent memory levels (ring entries, static slots) instead of a
// per-warp loop of them.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCtxThreads)
ctx_kernel(CtxParams p) {
  __shared__ uint32_t s_inst[kMaxCols];                // instruction of each column
  __shared__ float s_dyn[kMaxCols][kSlots - kStatic];  // its 9 dynamic slots, normalised
  __shared__ SubState s_st;                            // state after the apply step

  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
  const uint64_t s = blockIdx.x + p.first;
  if (s >= p.last) return;

  SubState* sp = p.state + s;
  const NormConsts& nc = *p.nc;
  Rings r{p.proc + s * (p.pmask + 1ull), p.wq + s * (p.wmask + 1ull), p.pmask, p.wmask, p.wmask + 1u};
  if (warp == 0) {
    SubState st = *sp;  // every lane holds a copy; lane 0 writes back
    uint32_t err = kOk;
    if (st.status == kOk) {
      if (st.has_pend) {
        const uint32_t F = st.pend_f;
        // fetch advance: K3 already moved cur by F (lumped); retire with budget bw*F
        if (F > 0) {
          if (p.per_cycle) {
            for (uint32_t c = 0; c < F && err == kOk; ++c) {
              st.cur += 1;
              warp_retire(st.cur, p.bw, r, st.ph, st.pt, st.wh, st.wt, &err);
            }
          } else {
            warp_retire(st.cur, static_cast<uint64_t>(p.bw) * F, r, st.ph, st.pt, st.wh, st.wt, &err);
          }
        }
        // forced stall (simcore.cpp:127-136): budget bw, not bw*gap
        while (err == kOk && st.pt - st.ph >= static_cast<uint32_t>(p.max_context)) {
          const uint32_t before = st.pt - st.ph;
          const RingEntry& h = r.proc[st.ph & r.pmask];
          const uint64_t gap = head_gap(st.cur, h.push, h.exec);
          st.cur += gap;
          st.overflow += gap;
          warp_retire(st.cur, p.bw, r, st.ph, st.pt, st.wh, st.wt, &err);
          if (err == kOk && st.pt - st.ph >= before) {
            err = kErrStall;
            st.err_tick = st.cur;
          }
        }
        if (err == kOk) {  // push (simcore.cpp:138-145)
          if (lane == 0) {
            RingEntry e;
            e.push = st.cur;
            e.idx = st.pos;
            e.exec = st.pend_e;
            e.store = st.pend_s;
            e.nexec = norm_slot(static_cast<int32_t>(st.pend_e), nc.mean[kSlotExecution], nc.sd[kSlotExecution]);
            e.nstore = norm_slot(static_cast<int32_t>(st.pend_s), nc.mean[kSlotStore], nc.sd[kSlotStore]);
            e.pc = st.t_pc;  // stashed by this sub-trace's previous gather (0 when none ran)
            e.addr = st.t_addr;
            e.flags = p.gather ? st.t_flags : p.iflags[st.begin + st.pos];
            r.proc[st.pt & r.pmask] = e;
          }
          st.pt += 1;
          st.pos += 1;
          st.has_pend = 0;
          if (st.pos == st.warm) {  // warm-up extension: counting starts after this step
            st.base_cur = st.cur;
            st.base_overflow = st.overflow;
          }
          // drain right after the last step (parallel.cpp:79, simcore.cpp:152-159)
          if (st.pos == st.len && st.count_drain) {
            while (err == kOk && (st.ph != st.pt || st.wh != st.wt)) {
              uint64_t gap = ~uint64_t{0};
              if (st.ph != st.pt) {
                const RingEntry& h = r.proc[st.ph & r.pmask];
                { const uint64_t g = head_gap(st.cur, h.push, h.exec); gap = g < gap ? g : gap; }
              }
              if (st.wh != st.wt) {
                const RingEntry& h = r.wq[st.wh & r.wmask];
                { const uint64_t g = head_gap(st.cur, h.push, h.store); gap = g < gap ? g : gap; }
              }
              if (gap < 1) gap = 1;
              st.cur += gap;
              st.drain += gap;
              const uint32_t ev = warp_retire(st.cur, p.bw, r, st.ph, st.pt, st.wh, st.wt, &err);
              if (err == kOk && ev == 0) {
                err = kErrDrain;
                st.err_tick = st.cur;
              }
            }
          }
        }
        if (err != kOk) st.status = err;
        __syncwarp();
        if (lane == 0) *sp = st;
        __syncwarp();
      }
    }
    (void)err;
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
  for (uint32_t c = tid; c <= ncols; c += kCtxThreads) {
    if (c == 0) {
      s_inst[0] = static_cast<uint32_t>(tgt);
#pragma unroll
      for (int k = kStatic; k < kSlots; ++k) s_dyn[0][k - kStatic] = nc.zero[k];
      continue;
    }
    const uint32_t j = c - 1;
    const RingEntry e = j < nproc ? r.proc[(st.pt - 1 - j) & r.pmask] : r.wq[(st.wt - 1 - (j - nproc)) & r.wmask];
    const int32_t res = static_cast<int32_t>(static_cast<uint32_t>(st.cur - e.push));
    // memory_dependency_flags (dataset.cpp:47-60)
    uint32_t f = (tpc / p.line) == (e.pc / p.line) ? 1u : 0u;
    if (tmem && (e.flags & kFlagMem)) {
      f |= (taddr == e.addr) ? 2u : 0u;
      f |= (taddr / p.line) == (e.addr / p.line) ? 4u : 0u;
      f |= (taddr / p.page) == (e.addr / p.page) ? 8u : 0u;
    }
    f |= (tpc / p.page) == (e.pc / p.page) ? 16u : 0u;
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
  for (uint32_t q0 = 0; q0 < n4; q0 += 4 * kCtxThreads) {
    float stv[4][4], dyv[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t jf = 4 * (q0 + u * kCtxThreads + tid) + t;
        const uint32_t col = jf / kSlots, slot = jf - col * kSlots;
        const uint32_t colc = jf < live ? col : 0u;
        const bool st_slot = slot < kStatic;
        stv[u][t] = __ldg(p.stat + static_cast<uint64_t>(s_inst[colc]) * kStatStride + (st_slot ? slot : 0u));
        dyv[u][t] = s_dyn[colc][st_slot ? 0u : slot - kStatic];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t q = q0 + u * kCtxThreads + tid;
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

// ---------------------------------------------------------------------------
// K3: hybrid decode (or truth in oracle mode) and the fetch-clock advance.
// ---------------------------------------------------------------------------
__global__ void decode_kernel(DecodeParams p) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x + p.first;
  if (s >= p.last) return;
  SubState* sp = p.state + s;
  if (sp->status != kOk) return;
  const uint32_t pos = sp->pos, len = sp->len;
  if (pos >= len) return;
  const uint64_t idx = sp->begin + pos;
  uint32_t t[3];
  if (p.truth) {
    t[0] = p.truth[3 * idx + 0];
    t[1] = p.truth[3 * idx + 1];
    t[2] = p.truth[3 * idx + 2];
  } else {
    const float* y = p.y + (s - p.first) * static_cast<uint64_t>(p.y_stride);
    decode_triple(y, *p.nc, p.class_fetch, p.class_exec, p.class_store,
                  (p.iflags[idx] & kFlagStore) != 0, t);
  }
  apply_decoded(sp, t, p.pred_fetch, p.per_cycle);
}

// Teacher-forced decode of caller logits (ilsim_gpu_predict).
__global__ void decode_only_kernel(const float* y, int y_stride, uint64_t n, const uint8_t* is_store,
                                   const NormConsts* nc, int cf, int ce, int cs, uint32_t* out) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  decode_triple(y + i * y_stride, *nc, cf, ce, cs, is_store[i] != 0, out + 3 * i);
}

// ---------------------------------------------------------------------------
// Pack: normalise the 41 static slots once per instruction and derive flags.
// ---------------------------------------------------------------------------
__global__ void pack_kernel(PackParams p) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
  if (i >= p.n) return;
  const uint32_t k = threadIdx.x;  // 0..63
  if (k < kStatic && p.stat) {
    int32_t raw;
    if (k < 13) raw = p.op[i * 13 + k];
    else if (k < 21) raw = p.src[i * 8 + (k - 13)];
    else if (k < 27) raw = p.dst[i * 6 + (k - 21)];
    else raw = p.hist[i * 14 + (k - 27)];
    p.stat[i * kStatStride + k] = norm_slot(raw, p.nc->mean[k], p.nc->sd[k]);
  } else if (k == 63) {
    const uint8_t ld = p.op[i * 13 + 1], stv = p.op[i * 13 + 2];
    p.iflags[i] = static_cast<uint8_t>(((ld | stv) ? kFlagMem : 0) | (stv ? kFlagStore : 0));
  }
}

__global__ void pack_inputs_kernel(const float* in, uint64_t n, uint32_t width, void* x, uint32_t x_stride,
                                   int x_bf16, uint64_t x_lo_off) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * width) return;
  const uint64_t smp = i / width;
  const uint32_t j = static_cast<uint32_t>(i - smp * width);
  if (x_bf16) {
    const uint32_t row = j / 100, within = j - 100 * row;
    static_cast<__nv_bfloat16*>(x)[smp * x_stride + row * 104 + within] = __float2bfloat16_rn(in[i]);
  } else if (x_lo_off) {
    const float v = in[i];
    const float h = __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xffffe000u);
    static_cast<float*>(x)[smp * x_stride + j] = h;
    static_cast<float*>(x)[smp * x_stride + j + x_lo_off] = v - h;
  } else {
    static_cast<float*>(x)[smp * x_stride + j] = in[i];
  }
}

void launch_pack_inputs(const float* in, uint64_t n, uint32_t width, void* x, uint32_t x_stride, int x_bf16,
                        uint64_t x_lo_off, cudaStream_t stream) {
  const uint64_t tot = n * width;
  if (tot == 0) return;
  pack_inputs_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, stream>>>(in, n, width, x, x_stride,
                                                                                    x_bf16, x_lo_off);
}

void launch_ctx(const CtxParams& p, cudaStream_t stream) {
  const uint64_t n = p.last - p.first;
  if (n == 0) return;
  launch_pdl(ctx_kernel, dim3(static_cast<unsigned>(n)), dim3(kCtxThreads), 0, stream, p);
}

void launch_decode(const DecodeParams& p, cudaStream_t stream) {
  const uint64_t n = p.last - p.first;
  if (n == 0) return;
  launch_pdl(decode_kernel, dim3(static_cast<unsigned>((n + 127) / 128)), dim3(128), 0, stream, p);
}

void launch_decode_only(const float* y, int y_stride, uint64_t n, const uint8_t* is_store,
                        const NormConsts* nc, int cf, int ce, int cs, uint32_t* out,
                        cudaStream_t stream) {
  if (n == 0) return;
  decode_only_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, stream>>>(
      y, y_stride, n, is_store, nc, cf, ce, cs, out);
}

void launch_pack(const PackParams& p, cudaStream_t stream) {
  if (p.n == 0) return;
  dim3 block(64, 4);
  pack_kernel<<<static_cast<unsigned>((p.n + 3) / 4), block, 0, stream>>>(p);
}

}  // namespace simnet
