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
#include "fc_decode.cuh"
#include "k1_device.cuh"
#include "launch.cuh"
#include "sim_kernels.cuh"

namespace simnet {


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
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = k1::lane_id();
  const uint64_t s = blockIdx.x + p.first;
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
  for (uint32_t c = tid; c <= ncols; c += kCtxThreads) {
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
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
  if (t >= p.n) return;
  const uint64_t i = p.seg_len ? p.seg_first + (t / p.seg_len) * p.seg_stride + t % p.seg_len : t;
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

// Test hook (ilsim_gpu_decode_outputs, path 1): the fused round's
// warp-cooperative decode (warp_decode_triple, one warp per sample, the label
// statistics in shared memory as the round front stages them).
__global__ void decode_warp_kernel(const float* y, int y_stride, uint64_t n, const uint8_t* is_store,
                                   const NormConsts* nc, int cf, int ce, int cs, uint32_t* out) {
  __shared__ double lab[6];
  if (threadIdx.x < 3) {
    lab[threadIdx.x] = nc->label_mean[threadIdx.x];
    lab[3 + threadIdx.x] = nc->label_sd[threadIdx.x];
  }
  __syncthreads();
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  uint32_t t[3];
  warp_decode_triple(y + i * y_stride, lab, cf, ce, cs, is_store[i] != 0, t);
  if ((threadIdx.x & 31) == 0) {
    out[3 * i + 0] = t[0];
    out[3 * i + 1] = t[1];
    out[3 * i + 2] = t[2];
  }
}

void launch_decode_warp(const float* y, int y_stride, uint64_t n, const uint8_t* is_store,
                        const NormConsts* nc, int cf, int ce, int cs, uint32_t* out,
                        cudaStream_t stream) {
  if (n == 0) return;
  decode_warp_kernel<<<static_cast<unsigned>((n + 3) / 4), 128, 0, stream>>>(y, y_stride, n, is_store, nc, cf,
                                                                             ce, cs, out);
}

// ---------------------------------------------------------------------------
// GPU trace ingest: a block stages 256 records (27,648 B) in shared memory with
// coalesced 16-B loads, then each thread extracts its record's fields
// (read_record, trace.cpp:64-83: address / size read as 0 without data).
// ---------------------------------------------------------------------------
constexpr int kRecBytes = 108, kRecPerBlock = 256;

__global__ void __launch_bounds__(kRecPerBlock) unpack_records_kernel(UnpackParams p) {
  __shared__ __align__(16) uint8_t srec[kRecPerBlock * kRecBytes];
  const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * kRecPerBlock;
  const uint64_t nrec = p.n - r0 < kRecPerBlock ? p.n - r0 : kRecPerBlock;
  const uint32_t bytes = static_cast<uint32_t>(nrec * kRecBytes);
  const uint8_t* src = p.rec + r0 * kRecBytes;  // 4-byte aligned (108 = 27 x 4)
  for (uint32_t i = threadIdx.x; i < bytes / 4; i += kRecPerBlock)
    reinterpret_cast<uint32_t*>(srec)[i] = __ldg(reinterpret_cast<const uint32_t*>(src) + i);
  __syncthreads();
  if (threadIdx.x >= nrec) return;
  const uint8_t* b = srec + threadIdx.x * kRecBytes;
  const uint64_t i = r0 + threadIdx.x;
  auto u16 = [&](int o) { return static_cast<uint16_t>(b[o] | (b[o + 1] << 8)); };
  auto u32 = [&](int o) { return static_cast<uint32_t>(u16(o)) | (static_cast<uint32_t>(u16(o + 2)) << 16); };
  auto u64 = [&](int o) { return static_cast<uint64_t>(u32(o)) | (static_cast<uint64_t>(u32(o + 4)) << 32); };
  p.pc[i] = u64(0);
#pragma unroll
  for (int k = 0; k < 13; ++k) p.op[i * 13 + k] = b[8 + k];
#pragma unroll
  for (int k = 0; k < 8; ++k) p.src[i * 8 + k] = u16(21 + 2 * k);
#pragma unroll
  for (int k = 0; k < 6; ++k) p.dst[i * 6 + k] = u16(37 + 2 * k);
  const bool has = b[49] != 0;
  p.addr[i] = has ? u64(50) : 0ull;
#pragma unroll
  for (int k = 0; k < 14; ++k) p.hist[i * 14 + k] = u16(60 + 2 * k);
  if (p.truth) {
#pragma unroll
    for (int k = 0; k < 3; ++k) p.truth[i * 3 + k] = u32(88 + 4 * k);
  }
}

void launch_unpack_records(const UnpackParams& p, cudaStream_t stream) {
  if (p.n == 0) return;
  unpack_records_kernel<<<static_cast<unsigned>((p.n + kRecPerBlock - 1) / kRecPerBlock), kRecPerBlock, 0, stream>>>(p);
}

void launch_pack(const PackParams& p, cudaStream_t stream) {
  if (p.n == 0) return;
  dim3 block(64, 4);
  pack_kernel<<<static_cast<unsigned>((p.n + 3) / 4), block, 0, stream>>>(p);
}

}  // namespace simnet
