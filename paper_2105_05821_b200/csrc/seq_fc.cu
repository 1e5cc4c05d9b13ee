// Persistent kernel for the FC-only predictor at small K (the sequential
// configuration c1: one sub-trace, K = 1): the whole simulation -- every round
// of K1 (apply + gather), K2 (FC1 -> ReLU -> FC2) and K3 (decode + clock) --
// is ONE cooperative launch (SURVEY.md §8(f) rank 1 for this predictor).
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
      const uint32_t e = i >> 1;
      uint64_t row;
      if (e < n)
        row = st.begin + proc_all[s * pcap + ((st.pt - 1 - e) & (pcap - 1))].idx;
      else
        row = st.begin + st.pos + (e - n);
      if (st.pos + (e >= n ? e - n : 0) >= st.len && e >= n) continue;
      const float* a = cx.stat + row * kStatStride + (i & 1) * 32;
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

bool seq_fc_fits(int flat, int hidden, int od, int K, int ctas, int pcap) {
  if (ctas < 2 || K < 1 || K > 8 || hidden < ctas - 1) return false;
  const size_t need = seq_fc_smem(flat, hidden, od, K, ctas, pcap) + sizeof(CtxSmem) + 8 * kFcMaxOut * 4 + 128;
  return need <= 227 * 1024;
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

}  // namespace simnet
