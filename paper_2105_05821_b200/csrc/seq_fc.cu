// Persistent kernels for the sequential configurations:
//   seq_fc_kernel  the FC-only predictor at K <= 2 (config c1: one sub-trace);
//   seq_c3_kernel  the C3 at one sub-trace (simulate_trace with the CNN), below.
// The whole simulation -- every round of K1 (apply + gather), K2 (the
// predictor) and K3 (decode + clock) -- is ONE cooperative launch.  For the
// FC-only predictor:
//
// A round of the launch-per-layer path is six dependent launches (ctx, two
// split-K GEMV pairs, decode), each a few microseconds of launch latency for
// microseconds of work.  Here the CTAs stay resident and the layers' weights
// stay in shared memory for the whole run:
//   CTA 0 (control): FC2 weights resident; per round: FC2 + decode of the
//     previous round's hidden layer, then K1 for its sub-traces (the same
//     ctx_one body as ctx_kernel), publishes the gathered rows (release flag);
//   CTAs 1..G-1 (workers): each keeps its slice of FC1's weights (a few hidden
//     units x all 5550 inputs, ~158 KB) in shared memory; per round: wait for
//     the rows (acquire), compute their hidden units, publish them (release
//     counter).
// Arithmetic order is exactly the split-K GEMV path's (sgemv_chunk_kernel /
// sgemv_reduce_kernel, gemm_simt.cu): per output, an fma chain over each
// 512-wide K chunk starting from 0, the chunk sums added in chunk order from
// 0, then bias (and ReLU for FC1); decode / apply as decode_kernel /
// ctx_kernel.  So results are bit-identical to the graph path.
//
// Every wait is bounded: a CTA that spins past ~4 s of polling raises the
// run's error flag and leaves (no hung GPU on a logic error).
#include <cuda_runtime.h>

#include <cstdlib>

#include "ctx_device.cuh"
#include "decode.cuh"
#include "fc_decode.cuh"
#include "gemm.cuh"
#include "host_util.cuh"
#include "seq_fc.cuh"

namespace simnet {

namespace {

constexpr int kSeqThreads = 256;
constexpr int kPad = kSgemmChunk + 1;  // padded chunk pitch of the staged rows (conflict-free)
constexpr uint32_t kExit = 0xffffffffu;

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr uint32_t kTraceRound = 100;

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Thread 0 polls until *p >= want (or kExit); bounded.  Returns the value seen.
__device__ uint32_t wait_at_least(const uint32_t* p, uint32_t want, uint32_t* err) {
  uint32_t v = ld_acquire(p);
  for (uint64_t spin = 0; v < want && v != kExit; ++spin) {
    if (spin > (1ull << 26)) {  // ~4 s of polling: a logic error, not a slow round
      atomicExch(err, 1u);
      return kExit;
    }
    if (spin > 64) __nanosleep(32);
    v = ld_acquire(p);
  }
  return v;
}

// Stage `rows` rows of `kdim` floats (row pitch `pitch` in global memory,
// written by another SM: L2 loads) as [row][chunk][kPad].
// 16-B loads (rows are 16-B aligned: pitch a multiple of 4 floats), all of a
// thread's loads of a block issued before its first store.
__device__ __forceinline__ void stage_rows(float* dst, const float* src, int rows, int kdim, uint64_t pitch,
                                           int nch) {
  constexpr int kBatch = 8;
  const int n4 = (kdim + 3) / 4;
  for (int r = 0; r < rows; ++r) {
    const float4* s4 = reinterpret_cast<const float4*>(src + r * pitch);
    for (int q0 = 0; q0 < n4; q0 += kBatch * kSeqThreads) {
      float4 v[kBatch];
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        const int q = q0 + i * kSeqThreads + threadIdx.x;
        v[i] = q < n4 ? __ldcg(s4 + q) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        const int k = 4 * (q0 + i * kSeqThreads + threadIdx.x);  // 4 | 512: a float4 never straddles chunks
        float* d = dst + (r * nch + k / kSgemmChunk) * kPad + k % kSgemmChunk;
        if (k < kdim) d[0] = v[i].x;
        if (k + 1 < kdim) d[1] = v[i].y;
        if (k + 2 < kdim) d[2] = v[i].z;
        if (k + 3 < kdim) d[3] = v[i].w;
      }
    }
  }
}

// Warm L1 with the static-slot rows the next gather will read (the current
// context entries' and the next target's, 192 B each; the trace is read-only,
// so the gather's __ldg hits them), while the control CTA waits on the workers.
__device__ __forceinline__ void prefetch_context(const CtxParams& cx, const SubState* st_all,
                                                 const RingEntry* proc_all, uint32_t pcap, int K) {
  for (int s = 0; s < K; ++s) {
    const SubState& st = st_all[s];
    const uint32_t n = st.pt - st.ph;
    const uint32_t lines = 2 * (n + 2);  // + the next two targets
    for (uint32_t i = threadIdx.x; i < lines; i += kSeqThreads) {
      const uint32_t e = i >> 1;  // entry e of the context (newest first), then the next two targets
      uint64_t row;
      if (e < n) {
        row = st.begin + proc_all[s * pcap + ((st.pt - 1 - e) & (pcap - 1))].idx;
      } else {
        const uint32_t pos = st.pos + (e - n);
        if (pos >= st.len) continue;  // past the sub-trace
        row = st.begin + pos;
      }
      const float* a = cx.stat + row * kStatStride + (i & 1) * 32;  // the row's two 128-B lines
      asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
    }
  }
}

// Chains: thread t < outs * nch owns (output t / nch, chunk t % nch); w is
// [kSgemmChunk][nchains] (step-major, conflict-free), x [row][chunk][kPad].
// part[row][t] = the chunk's fma chain from 0 (sgemv_chunk_kernel order).
__device__ __forceinline__ void chains(const float* w, const float* x, float* part, int rows, int nchains, int nch,
                                       int kdim) {
  const int t = threadIdx.x;
  if (t >= nchains) return;
  const int c = t % nch;
  const int len = min(kSgemmChunk, kdim - c * kSgemmChunk);
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (r * nch + c) * kPad;
    // the chain is serial (4-cycle FMA latency); unrolled 32 deep so each
    // block's 64 shared loads are in flight before its FMAs (a two-buffer
    // software pipeline of 16-step blocks measured slower: 3.1 -> 4.5 us)
    float acc = 0.0f;
    int j = 0;
    for (; j + 32 <= len; j += 32) {
      float xv[32], wv[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        xv[u] = xr[j + u];
        wv[u] = w[(j + u) * nchains + t];
      }
#pragma unroll
      for (int u = 0; u < 32; ++u) acc = fmaf(xv[u], wv[u], acc);
    }
    for (; j < len; ++j) acc = fmaf(xr[j], w[j * nchains + t], acc);
    part[r * nchains + t] = acc;
  }
}

}  // namespace

__global__ void __launch_bounds__(kSeqThreads, 1) seq_fc_kernel(SeqFcParams p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ CtxSmem csm;
  __shared__ uint32_t s_flag;
  const int tid = threadIdx.x;
  const int K = static_cast<int>(p.ctx.last - p.ctx.first);
  const int workers = gridDim.x - 1;

  if (blockIdx.x == 0) {
    // ------------------------------ control CTA ------------------------------
    __shared__ float ys[8 * kFcMaxOut];
    __shared__ double s_lab[6];
    const int warp = tid >> 5, lane = tid & 31;
    if (tid < 6) s_lab[tid] = tid < 3 ? p.dec.nc->label_mean[tid] : p.dec.nc->label_sd[tid - 3];
    const int nch = (p.hidden + kSgemmChunk - 1) / kSgemmChunk;
    const int nchains = p.od * nch;
    float* w2s = sm;                                           // [512][nchains]
    float* hs = w2s + kSgemmChunk * nchains;                   // [K][nch][kPad]
    float* part = hs + K * nch * kPad;                         // [K][nchains]
    // this CTA owns its sub-traces for the whole run: their SubStates and
    // processor-queue rings live in shared memory (generic pointers, so the K1
    // and K3 device code is unchanged); the write-queue rings stay in HBM
    const uint32_t pcap = p.ctx.pmask + 1;
    RingEntry* s_proc = reinterpret_cast<RingEntry*>(
        (reinterpret_cast<uintptr_t>(part + K * nchains) + 15) & ~uintptr_t{15});  // [K][pcap], 16-B aligned
    __shared__ SubState s_sub[8];
    for (int i = tid; i < K * static_cast<int>(sizeof(SubState) / 4); i += kSeqThreads)
      reinterpret_cast<uint32_t*>(s_sub)[i] = reinterpret_cast<const uint32_t*>(p.ctx.state + p.ctx.first)[i];
    CtxParams cx = p.ctx;
    cx.state = s_sub - p.ctx.first;
    cx.proc = s_proc - p.ctx.first * pcap;
    SubState* dstate = s_sub - p.dec.first;
    for (int i = tid; i < kSgemmChunk * nchains; i += kSeqThreads) {
      const int j = i / nchains, t = i % nchains, o = t / nch, c = t % nch, k = c * kSgemmChunk + j;
      w2s[i] = k < p.hidden ? p.w2[static_cast<uint64_t>(k) * p.od + o] : 0.0f;
    }
    __syncthreads();
    for (uint32_t r = 0; r <= p.rounds; ++r) {
      long long* tr = (p.trace && r == kTraceRound && tid == 0) ? p.trace : nullptr;
      if (r > 0) {
        // FC2 + decode of round r-1 (sgemv pair order, then decode_kernel)
        if (tr) tr[0] = gtimer();
        if (cx.gather) prefetch_context(cx, s_sub, s_proc, pcap, K);
        if (tid == 0) s_flag = wait_at_least(p.flags + 1, r * static_cast<uint32_t>(workers), p.flags + 2);
        __syncthreads();
        if (s_flag == kExit) break;
        if (tr) tr[1] = gtimer();
        stage_rows(hs, p.h, K, p.hidden, p.hidden, nch);
        __syncthreads();
        if (tr) tr[2] = gtimer();
        chains(w2s, hs, part, K, nchains, nch, p.hidden);
        __syncthreads();
        if (tr) tr[3] = gtimer();
        for (int i = tid; i < K * p.od; i += kSeqThreads) {
          const int s = i / p.od, o = i % p.od;
          float tot = 0.0f;
          for (int c = 0; c < nch; ++c) tot += part[s * nchains + o * nch + c];
          ys[s * kFcMaxOut + o] = tot + p.b2[o];
        }
        __syncthreads();
        if (warp < K) {  // K3 (decode_kernel's decode_triple + apply_decoded): warp w, sub-trace w,
                         // the three heads on lanes 0-2 (warp_decode_triple, the fused rounds' form)
          SubState* sp = dstate + p.dec.first + warp;
          SubState st = *sp;
          if (st.status == kOk && st.pos < st.len) {
            uint32_t t3[3];
            // t_flags: the target's flags, stashed by the gather (ctx_one) that built this input
            warp_decode_triple(ys + warp * kFcMaxOut, s_lab, p.dec.class_fetch, p.dec.class_exec,
                               p.dec.class_store, (st.t_flags & kFlagStore) != 0, t3);
            apply_decoded_reg(st, t3, p.dec.pred_fetch, p.dec.per_cycle);
            __syncwarp();  // every lane has read *sp (shared memory) before lane 0 rewrites it
            if (lane == 0) *sp = st;
          }
        }
        __syncthreads();
      }
      if (tr) tr[4] = gtimer();
      // K1: apply the decoded step, gather the next rows (the last pass: apply + drain only)
      CtxParams cp = cx;
      cp.gather = r < p.rounds ? p.ctx.gather : 0;
      for (uint64_t s = cp.first; s < cp.last; ++s) {
        ctx_one<kSeqThreads>(cp, s, csm);
        __syncthreads();
      }
      if (r == p.rounds) break;
      if (tr) tr[5] = gtimer();
      __threadfence();  // this thread's row stores, before the release below
      __syncthreads();
      if (tid == 0) st_release(p.flags, r + 1);
      if (tr) tr[6] = gtimer();
    }
    __syncthreads();
    if (tid == 0) st_release(p.flags, kExit);
    for (int i = tid; i < K * static_cast<int>(sizeof(SubState) / 4); i += kSeqThreads)
      reinterpret_cast<uint32_t*>(p.ctx.state + p.ctx.first)[i] = reinterpret_cast<const uint32_t*>(s_sub)[i];
    return;
  }

  // ------------------------------ worker CTAs ------------------------------
  const int wid = blockIdx.x - 1;
  const int o0 = static_cast<int>(static_cast<int64_t>(p.hidden) * wid / workers);
  const int o1 = static_cast<int>(static_cast<int64_t>(p.hidden) * (wid + 1) / workers);
  const int outs = o1 - o0;
  const int nch = (p.flat + kSgemmChunk - 1) / kSgemmChunk;
  const int nchains = outs * nch;
  const int cmax = p.max_outs * nch;
  float* w1s = sm;                          // [512][nchains]
  float* xs = w1s + kSgemmChunk * cmax;     // [K][nch][kPad]
  float* part = xs + K * nch * kPad;        // [K][nchains]
  for (int i = tid; i < kSgemmChunk * nchains; i += kSeqThreads) {
    const int j = i / nchains, t = i % nchains, o = o0 + t / nch, c = t % nch, k = c * kSgemmChunk + j;
    w1s[i] = k < p.flat ? p.w1[static_cast<uint64_t>(k) * p.hidden + o] : 0.0f;
  }
  __syncthreads();
  for (uint32_t r = 0;; ++r) {
    long long* tr = (p.trace && r == kTraceRound && tid == 0 && blockIdx.x == 1) ? p.trace + 8 : nullptr;
    if (tr) tr[0] = gtimer();
    if (tid == 0) s_flag = wait_at_least(p.flags, r + 1, p.flags + 2);
    __syncthreads();
    if (s_flag == kExit) break;
    if (tr) tr[1] = gtimer();
    stage_rows(xs, static_cast<const float*>(p.ctx.x), K, p.flat, p.ctx.x_stride, nch);
    __syncthreads();
    if (tr) tr[2] = gtimer();
    chains(w1s, xs, part, K, nchains, nch, p.flat);
    __syncthreads();
    if (tr) tr[3] = gtimer();
    for (int i = tid; i < K * outs; i += kSeqThreads) {
      const int s = i / outs, ol = i % outs;
      float tot = 0.0f;
      for (int c = 0; c < nch; ++c) tot += part[s * nchains + ol * nch + c];
      p.h[static_cast<uint64_t>(s) * p.hidden + o0 + ol] = fmaxf(tot + p.b1[o0 + ol], 0.0f);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(p.flags + 1, 1u);  // after the fence: the hidden units are visible
    if (tr) tr[4] = gtimer();
  }
}

size_t seq_fc_smem(int flat, int hidden, int od, int K, int ctas, int pcap) {
  const int workers = ctas - 1;
  const int max_outs = (hidden + workers - 1) / workers;
  const int nch1 = (flat + kSgemmChunk - 1) / kSgemmChunk, nch2 = (hidden + kSgemmChunk - 1) / kSgemmChunk;
  const size_t worker = (static_cast<size_t>(kSgemmChunk) * max_outs * nch1 + static_cast<size_t>(K) * nch1 * kPad +
                         static_cast<size_t>(K) * max_outs * nch1) * 4;
  const size_t control = (static_cast<size_t>(kSgemmChunk) * od * nch2 + static_cast<size_t>(K) * nch2 * kPad +
                          static_cast<size_t>(K) * od * nch2) * 4 + 16 +
                         static_cast<size_t>(K) * pcap * sizeof(RingEntry);
  return worker > control ? worker : control;
}

// A cooperative grid of `ctas` CTAs must be co-resident: one per SM needs the
// shared memory (and nothing else on the device holding the SMs, e.g. MPS
// clients).  When the occupancy query says no, the caller takes the
// launch-per-layer rounds instead.
bool coresident(const void* kernel, int threads, size_t smem, int ctas) {
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int per_sm = 0, dev = 0, sms = 0, coop = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess ||
      cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return coop != 0 && per_sm * sms >= ctas;
}

bool seq_fc_fits(int flat, int hidden, int od, int K, int ctas, int pcap) {
  if (ctas < 2 || K < 1 || K > 8 || hidden < ctas - 1) return false;
  const size_t smem = seq_fc_smem(flat, hidden, od, K, ctas, pcap);
  const size_t need = smem + sizeof(CtxSmem) + 8 * kFcMaxOut * 4 + 128;
  return need <= 227 * 1024 && coresident(reinterpret_cast<const void*>(seq_fc_kernel), kSeqThreads, smem, ctas);
}

void launch_seq_fc(SeqFcParams p, int ctas, cudaStream_t s) {
  const int K = static_cast<int>(p.ctx.last - p.ctx.first);
  p.max_outs = (p.hidden + ctas - 2) / (ctas - 1);
  const size_t smem = seq_fc_smem(p.flat, p.hidden, p.od, K, ctas, static_cast<int>(p.ctx.pmask + 1));
  CUDA_OK(cudaFuncSetAttribute(seq_fc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  void* args[] = {&p};
  CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(seq_fc_kernel), dim3(ctas), dim3(kSeqThreads), args,
                                      smem, s));
}

// ---------------------------------------------------------------------------
// The C3 at one sub-trace (simulate_trace with the CNN, fp32): the same
// persistent structure.  The control CTA keeps the three conv layers' and FC2's
// weights, the sub-trace state, its processor-queue ring AND the gathered input
// row in shared memory, so per round it runs K1 (ctx_one writes the row into
// shared memory), conv0 -> conv1 -> conv2, publishes the 1,024-float flat
// output, and after the workers' FC1 runs FC2 + decode.  Worker CTAs keep FC1's
// weight columns for their hidden units.  Every layer is the reference's order
// (oracle/cnn_restated.cpp gemm_cm): one fma chain per output, k ascending,
// then bias and ReLU -- bit-identical to the fp32 SIMT rounds.
// ---------------------------------------------------------------------------
namespace {

constexpr int kC3C = 64;  // channels of every C3 conv layer

// One conv layer on the control CTA: out[j][o] = ReLU(chain_k W[k][o] * in[j][k] + b[o]),
// in = [npos][kdim] (the previous layer's [2 npos][64] viewed as [npos][128]),
// W = [kdim][64] (reference column-major).  Thread t: channel t % 64, positions
// (t / 64) + 4 i, taken four at a time (four independent chains; k in steps of
// 4, 16-B loads of the input rows).  Positions >= live have an all-+0 input
// (conv0: columns past the context): their chain is +0 exactly, so their
// output is ReLU(+0 + b) without the loop.  (Also skipping conv1 / conv2 rows
// built only from such rows, computing their shared value once, measured
// slower: the single serial chain it adds outweighs the rows it saves.)
template <int kPos>
__device__ __forceinline__ void conv_layer(const float* in, int kdim, const float* w, const float* b, float* out,
                                           int live) {
  const int o = threadIdx.x % kC3C, pg = threadIdx.x / kC3C;
  constexpr int kPer = kPos / 4;
  const float bo = b[o];
#pragma unroll 1
  for (int ib = 0; ib < kPer; ib += 4) {
    if (pg + 4 * ib >= live) {  // warp-uniform: the rest of this thread's positions are dead
      for (int i = ib; i < kPer; ++i) out[(pg + 4 * i) * kC3C + o] = fmaxf(0.0f + bo, 0.0f);
      break;
    }
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    const float* r0 = in + (pg + 4 * ib) * kdim;
#pragma unroll 2
    for (int k = 0; k < kdim; k += 4) {
      const float w0 = w[(k + 0) * kC3C + o], w1 = w[(k + 1) * kC3C + o];
      const float w2 = w[(k + 2) * kC3C + o], w3 = w[(k + 3) * kC3C + o];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 x = *reinterpret_cast<const float4*>(r0 + 4 * i * kdim + k);
        acc[i] = fmaf(w0, x.x, acc[i]);
        acc[i] = fmaf(w1, x.y, acc[i]);
        acc[i] = fmaf(w2, x.z, acc[i]);
        acc[i] = fmaf(w3, x.w, acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) out[(pg + 4 * (ib + i)) * kC3C + o] = fmaxf(acc[i] + bo, 0.0f);
  }
}

}  // namespace

__global__ void __launch_bounds__(kSeqThreads, 1) seq_c3_kernel(SeqC3Params p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ CtxSmem csm;
  __shared__ uint32_t s_flag;
  __shared__ __align__(16) SubState s_sub[1];
  const int tid = threadIdx.x;
  const int workers = gridDim.x - 1;

  if (blockIdx.x == 0) {
    // ------------------------------ control CTA ------------------------------
    __shared__ double s_lab[6];
    __shared__ float ys[kFcMaxOut];
    const int warp = tid >> 5, lane = tid & 31;
    if (tid < 6) s_lab[tid] = tid < 3 ? p.dec.nc->label_mean[tid] : p.dec.nc->label_sd[tid - 3];
    float* w0 = sm;                        // [100][64]
    float* w1 = w0 + 100 * kC3C;           // [128][64]
    float* w2 = w1 + 128 * kC3C;           // [128][64]
    float* bs = w2 + 128 * kC3C;           // b0 | b1 | b2 (3 x 64)
    float* w2f = bs + 3 * kC3C;            // FC2 [hidden][od]
    float* x = w2f + p.hidden * p.od + ((4 - (p.hidden * p.od) % 4) % 4);  // [128 columns][50], 16-B aligned
    float* a0 = x + 128 * kSlots;          // [64][64]
    float* a1 = a0 + 64 * kC3C;            // [32][64]
    float* a2 = a1 + 32 * kC3C;            // [16][64] = flat
    float* hs = a2 + 16 * kC3C;            // [hidden]
    RingEntry* s_proc = reinterpret_cast<RingEntry*>(hs + ((p.hidden + 3) & ~3));  // [pcap]
    const uint32_t pcap = p.ctx.pmask + 1;
    for (int i = tid; i < 100 * kC3C; i += kSeqThreads) w0[i] = p.w0[i];
    for (int i = tid; i < 128 * kC3C; i += kSeqThreads) w1[i] = p.w1c[i];
    for (int i = tid; i < 128 * kC3C; i += kSeqThreads) w2[i] = p.w2c[i];
    for (int i = tid; i < 3 * kC3C; i += kSeqThreads) bs[i] = (i < kC3C ? p.b0 : (i < 2 * kC3C ? p.b1c : p.b2c))[i % kC3C];
    for (int i = tid; i < p.hidden * p.od; i += kSeqThreads) w2f[i] = p.w2f[i];
    for (int i = tid; i < 128 * kSlots; i += kSeqThreads) x[i] = 0.0f;  // padding columns stay +0
    for (int i = tid; i < static_cast<int>(sizeof(SubState) / 4); i += kSeqThreads)
      reinterpret_cast<uint32_t*>(s_sub)[i] = reinterpret_cast<const uint32_t*>(p.ctx.state + p.ctx.first)[i];
    CtxParams cx = p.ctx;
    cx.state = s_sub - p.ctx.first;
    cx.proc = s_proc - p.ctx.first * pcap;
    cx.x = x;  // the gathered row goes to shared memory
    cx.x_full = 0;
    __syncthreads();
    for (uint32_t r = 0; r <= p.rounds; ++r) {
      long long* tr = (p.trace && r == kTraceRound && tid == 0) ? p.trace : nullptr;
      if (r > 0) {
        // FC2 + decode of round r-1
        if (tr) tr[0] = gtimer();
        prefetch_context(cx, s_sub, s_proc, pcap, 1);
        if (tid == 0) s_flag = wait_at_least(p.flags + 1, r * static_cast<uint32_t>(workers), p.flags + 2);
        __syncthreads();
        if (s_flag == kExit) break;
        if (tr) tr[1] = gtimer();
        for (int i = tid; i < p.hidden; i += kSeqThreads) hs[i] = __ldcg(p.h + i);
        __syncthreads();
        if (tid < p.od) {
          float y = 0.0f;
#pragma unroll 8
          for (int k = 0; k < p.hidden; ++k) y = fmaf(w2f[k * p.od + tid], hs[k], y);
          ys[tid] = y + p.b2f[tid];
        }
        __syncthreads();
        if (tr) tr[2] = gtimer();
        if (warp == 0) {
          SubState st = s_sub[0];
          if (st.status == kOk && st.pos < st.len) {
            uint32_t t3[3];
            warp_decode_triple(ys, s_lab, p.dec.class_fetch, p.dec.class_exec, p.dec.class_store,
                               (st.t_flags & kFlagStore) != 0, t3);
            apply_decoded_reg(st, t3, p.dec.pred_fetch, p.dec.per_cycle);
            __syncwarp();
            if (lane == 0) s_sub[0] = st;
          }
        }
        __syncthreads();
      }
      if (tr) tr[3] = gtimer();
      CtxParams cp = cx;
      cp.gather = r < p.rounds ? 1 : 0;
      ctx_one<kSeqThreads>(cp, cp.first, csm);
      __syncthreads();
      if (r == p.rounds) break;
      if (tr) tr[4] = gtimer();
      if (s_sub[0].status != kOk || s_sub[0].pos >= s_sub[0].len) {
        // nothing was gathered (an error): publish anyway so the workers' round count stays in step
      } else {
        const int live = static_cast<int>(s_sub[0].xcols + 1) / 2;  // conv0 positions with a live column
        conv_layer<64>(x, 100, w0, bs, a0, live);
        __syncthreads();
        if (tr) tr[5] = gtimer();
        conv_layer<32>(a0, 128, w1, bs + kC3C, a1, 32);
        __syncthreads();
        conv_layer<16>(a1, 128, w2, bs + 2 * kC3C, a2, 16);
        __syncthreads();
        if (tr) tr[6] = gtimer();
      }
      for (int i = tid; i < 16 * kC3C; i += kSeqThreads) p.flat[i] = a2[i];
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(p.flags, r + 1);
      if (tr) tr[7] = gtimer();
    }
    __syncthreads();
    if (tid == 0) st_release(p.flags, kExit);
    for (int i = tid; i < static_cast<int>(sizeof(SubState) / 4); i += kSeqThreads)
      reinterpret_cast<uint32_t*>(p.ctx.state + p.ctx.first)[i] = reinterpret_cast<const uint32_t*>(s_sub)[i];
    return;
  }

  // ------------------------------ worker CTAs: FC1 ------------------------------
  const int wid = blockIdx.x - 1;
  const int o0 = static_cast<int>(static_cast<int64_t>(p.hidden) * wid / workers);
  const int o1 = static_cast<int>(static_cast<int64_t>(p.hidden) * (wid + 1) / workers);
  const int outs = o1 - o0;
  float* w1s = sm;                 // [1024][outs]
  float* fs = w1s + 1024 * 4;      // flat [1024]
  for (int i = tid; i < 1024 * outs; i += kSeqThreads) {
    const int k = i / outs, ol = i % outs;
    w1s[i] = p.w1f[static_cast<uint64_t>(k) * p.hidden + o0 + ol];
  }
  __syncthreads();
  for (uint32_t r = 0;; ++r) {
    long long* tr = (p.trace && r == kTraceRound && tid == 0 && blockIdx.x == 1) ? p.trace + 8 : nullptr;
    if (tid == 0) s_flag = wait_at_least(p.flags, r + 1, p.flags + 2);
    __syncthreads();
    if (s_flag == kExit) break;
    if (tr) tr[0] = gtimer();
    for (int i = tid; i < 1024 / 4; i += kSeqThreads)
      reinterpret_cast<float4*>(fs)[i] = __ldcg(reinterpret_cast<const float4*>(p.flat) + i);
    __syncthreads();
    if (tid < outs) {  // one chain over K = 1024 (the reference's order), 32 loads in flight per block
      float acc = 0.0f;
      for (int k = 0; k < 1024; k += 32) {
        float xv[32], wv[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          xv[u] = fs[k + u];
          wv[u] = w1s[(k + u) * outs + tid];
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) acc = fmaf(wv[u], xv[u], acc);
      }
      p.h[o0 + tid] = fmaxf(acc + p.b1f[o0 + tid], 0.0f);
    }
    if (tr) tr[1] = gtimer();
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(p.flags + 1, 1u);
    if (tr) tr[2] = gtimer();
  }
}

size_t seq_c3_smem(int hidden, int od, int pcap) {
  const size_t control = (static_cast<size_t>(100 + 128 + 128) * kC3C + 3 * kC3C + static_cast<size_t>(hidden) * od +
                          4 + 128 * kSlots + (64 + 32 + 16) * kC3C + ((hidden + 3) & ~3)) * 4 +
                         static_cast<size_t>(pcap) * sizeof(RingEntry) + 16;
  const size_t worker = (1024 * 4 + 1024) * 4;
  return control > worker ? control : worker;
}

bool seq_c3_fits(int hidden, int od, int ctas, int pcap) {
  if (ctas < 2 || od > kFcMaxOut || (hidden + ctas - 2) / (ctas - 1) > 4) return false;
  const size_t smem = seq_c3_smem(hidden, od, pcap);
  return smem + sizeof(CtxSmem) + 1024 <= 227 * 1024 &&
         coresident(reinterpret_cast<const void*>(seq_c3_kernel), kSeqThreads, smem, ctas);
}

void launch_seq_c3(SeqC3Params p, int ctas, cudaStream_t s) {
  const size_t smem = seq_c3_smem(p.hidden, p.od, static_cast<int>(p.ctx.pmask + 1));
  CUDA_OK(cudaFuncSetAttribute(seq_c3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  void* args[] = {&p};
  CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(seq_c3_kernel), dim3(ctas), dim3(kSeqThreads), args,
                                      smem, s));
}

}  // namespace simnet
