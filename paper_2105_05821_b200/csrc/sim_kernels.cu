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
#include "ctx_device.cuh"

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
  __shared__ CtxSmem sm;
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  ctx_one<kCtxThreads>(p, blockIdx.x + p.first, sm);
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
