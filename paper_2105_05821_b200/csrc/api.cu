// Host driver behind include/ilsim_gpu.h: validation with the reference's
// error texts, partition / sharding, device layout, the round loop (CUDA
// graphs of K1 -> K2 -> K3 per round), result collection.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ilsim_gpu.h"
#include "common.cuh"
#include "conv_chain.cuh"
#include "gemm.cuh"
#include "host_util.cuh"
#include "model.cuh"
#include "seq_fc.cuh"
#include "sim_kernels.cuh"

using namespace simnet;

namespace {

uint32_t next_pow2(uint32_t v) {
  uint32_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

std::vector<uint64_t> partition_starts(uint64_t n, uint64_t k) {  // parallel.cpp:9-24
  if (k < 1 || k > std::max<uint64_t>(n, 1))
    throw ApiError("sub-trace count " + std::to_string(k) + " out of range for trace of " +
                   std::to_string(n));
  std::vector<uint64_t> s(k);
  const uint64_t base = n / k, rem = n % k;
  uint64_t at = 0;
  for (uint64_t i = 0; i < k; ++i) {
    s[i] = at;
    at += base + (i < rem ? 1 : 0);
  }
  return s;
}

// Sub-trace count per parallel.cpp:28-41 (the sequential driver is K=1).
uint64_t derive_k(const ilsim_sim_config& c, uint64_t n) {
  if (c.sequential) return 1;
  uint64_t k = c.k;
  if (c.subtrace_size > 0) {
    const uint64_t derived = n == 0 ? 1 : (n + c.subtrace_size - 1) / c.subtrace_size;
    if (k == 0)
      k = derived;
    else if (k != derived)
      throw ApiError("inconsistent partition: k=" + std::to_string(k) + " but subtrace size " +
                     std::to_string(c.subtrace_size) + " implies k=" + std::to_string(derived));
  }
  if (k == 0) k = 1;
  if (c.batch_max == 0) throw ApiError("batch_max must be >= 1");
  return k;
}

struct Plan {
  uint64_t n = 0, k = 0, sb = 0, se = 0;  // trace length, sub-traces, shard range
  std::vector<uint64_t> starts;
  uint64_t g0 = 0, g1 = 0;                 // device trace slice [g0, g1)
  uint64_t own0 = 0, own1 = 0;             // owned instructions of the shard
};

Plan make_plan(const ilsim_sim_config& c, uint64_t n) {
  Plan p;
  p.n = n;
  p.k = derive_k(c, n);
  if (n == 0) return p;
  p.starts = partition_starts(n, p.k);
  p.sb = c.shard_begin;
  p.se = c.shard_end;
  if (p.sb == 0 && p.se == 0) p.se = p.k;
  if (p.sb >= p.se || p.se > p.k) throw ApiError("invalid shard range");
  auto end_of = [&](uint64_t i) { return i + 1 < p.k ? p.starts[i + 1] : n; };
  p.own0 = p.starts[p.sb];
  p.own1 = end_of(p.se - 1);
  p.g0 = p.own0 - std::min<uint64_t>(c.warmup, p.own0);
  p.g1 = p.own1;
  return p;
}

// Row of the view's arrays that holds global instruction P.g0 (the view may
// hold only a slice [base, ...) of the global trace, ilsim_trace_view.base).
uint64_t view_row(const ilsim_trace_view* t, const Plan& P) {
  if (t->base > P.g0 || t->base > t->n)
    throw ApiError("trace view (base " + std::to_string(t->base) + ") does not cover the shard's first instruction " +
                   std::to_string(P.g0));
  return P.g0 - t->base;
}

}  // namespace

struct ilsim_gpu_ctx {
  int device = 0;
  int precision = ILSIM_PREC_FP32;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8] = {};
  std::string err;

  // model
  bool has_model = false;
  ilsim_cnn_config cfg{};
  std::vector<double> norm;
  DevModel model;
  NormConsts nc_host{};
  DevBuf nc_dev;
  uint64_t model_gen = 0;

  // trace (device slice [g0, g1) of a trace of t_total instructions)
  bool has_trace = false;
  uint64_t t_total = 0, g0 = 0, g1 = 0;
  bool has_truth = false;
  uint64_t packed_gen = ~0ull;  // model_gen the static table was packed with
  DevBuf pc, addr, op, src, dst, hist, truth, stat, iflags;

  // run buffers
  DevBuf state, proc, wq, x, y, act, pred_fetch;
  DevBuf rec_stage;  // SNT1 record staging for the GPU trace ingest
  DevBuf seq_flags;  // persistent FC kernel: publish / count / error words

  // simulate_parallel with the trace upload overlapped with the rounds: the
  // borrowed host view, uploaded window by window on copy_stream
  const ilsim_trace_view* deferred = nullptr;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> win_ev;

  // capture hook
  uint32_t cap_round = UINT32_MAX;
  float* cap_host = nullptr;
  uint64_t cap_rows = 0;
};

namespace {

void set_norm(ilsim_gpu_ctx* c, const double* norm) {
  NormConsts& h = c->nc_host;
  for (int k = 0; k < kSlots; ++k) {
    h.mean[k] = norm ? norm[k] : 0.0;
    h.sd[k] = norm ? norm[50 + k] : 1.0;
    h.zero[k] = norm_slot(0, h.mean[k], h.sd[k]);
    h.one[k] = norm_slot(1, h.mean[k], h.sd[k]);
  }
  for (int j = 0; j < 3; ++j) {
    h.label_mean[j] = norm ? norm[100 + j] : 0.0;
    h.label_sd[j] = norm ? norm[103 + j] : 1.0;
  }
  c->nc_dev.need(sizeof(NormConsts));
  CUDA_OK(cudaMemcpy(c->nc_dev.p, &h, sizeof(NormConsts), cudaMemcpyHostToDevice));
}

template <typename T>
void upload(DevBuf& b, const T* src, uint64_t count, cudaStream_t s) {
  b.need(count * sizeof(T));
  if (count) CUDA_OK(cudaMemcpyAsync(b.p, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
}

// Effective max_context for a run (cmd_simulate: the model's, ilsim_main.cpp:141).
int effective_mc(const ilsim_gpu_ctx* c, const ilsim_sim_config& cfg) {
  if (cfg.max_context > 0) return cfg.max_context;
  return c->has_model ? c->cfg.max_context : 110;
}

void pack_if_needed(ilsim_gpu_ctx* c, bool needs_input) {
  const uint64_t n = c->g1 - c->g0;
  if (c->packed_gen == c->model_gen && (!needs_input || c->stat.bytes >= n * kStatStride * 4)) return;
  PackParams pp{};
  pp.n = n;
  pp.op = c->op.as<uint8_t>();
  pp.src = c->src.as<uint16_t>();
  pp.dst = c->dst.as<uint16_t>();
  pp.hist = c->hist.as<uint16_t>();
  pp.nc = c->nc_dev.as<NormConsts>();
  pp.stat = needs_input ? static_cast<float*>(c->stat.need(n * kStatStride * sizeof(float))) : nullptr;
  pp.iflags = static_cast<uint8_t*>(c->iflags.need(n));
  launch_pack(pp, c->stream);
  CUDA_OK(cudaGetLastError());
  if (needs_input) c->packed_gen = c->model_gen;
}

void run_impl(ilsim_gpu_ctx* c, const ilsim_sim_config& cfg, ilsim_sub_result* subs, uint64_t sub_cap,
              uint32_t* predicted_fetch, ilsim_totals* tot) {
  if (!c->has_trace) throw ApiError("no trace loaded");
  const uint64_t n = c->t_total;
  const bool oracle = cfg.oracle != 0;
  const bool needs_input = !oracle || cfg.reserved[1] != 0;
  const Plan P = make_plan(cfg, n);
  const int mc = effective_mc(c, cfg);
  std::memset(tot, 0, sizeof(*tot));

  if (n == 0) {  // parallel.cpp:44-50 / simcore.cpp:167-174: one empty result
    if (sub_cap < 1) throw ApiError("sub_cap too small");
    subs[0] = ilsim_sub_result{0, 0, 0, 0, 0, 0, 1};
    tot->sub_traces = 1;
    return;
  }
  // SimCore ctor checks (simcore.cpp:13-18)
  if (mc < 1) throw ApiError("max_context must be >= 1");
  if (cfg.retire_bandwidth < 1) throw ApiError("retire_bandwidth must be >= 1");
  if (needs_input && !c->has_model)
    throw ApiError("predictor requires inputs but provides no normalization stats");
  if (oracle && !c->has_truth) throw ApiError("oracle mode requires truth latencies");
  if (needs_input && !oracle && mc != c->cfg.max_context) throw ApiError("max_context differs from the model's");
  if (needs_input && mc + 1 > kMaxCols) throw ApiError("max_context too large for the GPU gather");
  if (P.g0 != c->g0 || P.g1 != c->g1) throw ApiError("loaded trace slice does not match this configuration");

  const uint64_t K = P.se - P.sb;
  if (K > sub_cap) throw ApiError("sub_cap too small");
  const uint32_t pcap = next_pow2(static_cast<uint32_t>(mc));
  // write ring: explicit, or auto = 2048 entries capped by the longest
  // sub-trace (its write queue never holds more stores than it has
  // instructions), so 1M short sub-traces do not reserve 96 KB each; an auto
  // ring that overflows is regrown (run_growing_ring)

  // per-sub-trace initial state
  std::vector<SubState> hs(K);
  uint32_t rounds = 0;
  for (uint64_t j = 0; j < K; ++j) {
    const uint64_t i = P.sb + j;
    const uint64_t s = P.starts[i];
    const uint64_t e = i + 1 < P.k ? P.starts[i + 1] : n;
    const uint64_t w = std::min<uint64_t>(cfg.warmup, s);
    SubState& st = hs[j];
    std::memset(&st, 0, sizeof(st));
    st.begin = s - w - P.g0;
    st.len = static_cast<uint32_t>(e - s + w);
    st.warm = static_cast<uint32_t>(w);
    st.fetch_off = s - P.own0;
    st.count_drain = (cfg.drain_trim && i + 1 < P.k) ? 0u : 1u;
    rounds = std::max(rounds, st.len);
  }
  const uint32_t wcap =
      next_pow2(cfg.write_ring > 0 ? static_cast<uint32_t>(cfg.write_ring) : std::min<uint32_t>(2048u, rounds + 1u));
  // Overlapped upload (simulate_parallel): round r reads trace position r of
  // every sub-trace (and older ones), so the trace goes up in windows of
  // positions, each copied (2-D copies over runs of equal-length sub-traces)
  // and packed on copy_stream while earlier windows' rounds run.
  uint32_t win_rounds = 0, n_win = 0;
  if (c->deferred) {
    win_rounds = std::max<uint32_t>(16, ((rounds + 15) / 16 + 15) / 16 * 16);
    if (const char* e = std::getenv("SIMNET_WIN_ROUNDS"))  // A/B: window size in rounds
      win_rounds = std::max<uint32_t>(16, static_cast<uint32_t>(std::atoi(e)) / 16 * 16);
    n_win = (rounds + win_rounds - 1) / win_rounds;
    struct Group { uint64_t first_begin, stride, count; uint32_t len; };
    std::vector<Group> groups;
    for (uint64_t j = 0; j < K; ++j) {
      const SubState& st = hs[j];
      if (!groups.empty()) {
        Group& g = groups.back();
        const uint64_t stride = g.count == 1 ? st.begin - g.first_begin : g.stride;
        if (st.len == g.len && st.begin == g.first_begin + g.count * stride && stride >= win_rounds) {
          g.stride = stride;
          ++g.count;
          continue;
        }
      }
      groups.push_back(Group{st.begin, static_cast<uint64_t>(win_rounds), 1, st.len});
    }
    while (c->win_ev.size() < n_win) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->win_ev.push_back(e);
    }
    const ilsim_trace_view* t = c->deferred;
    const uint64_t row0 = view_row(t, P);
    auto copy2d = [&](void* dev, const void* host, size_t esz, const Group& g, uint64_t p0, uint64_t len) {
      const size_t pitch = g.stride * esz, width = len * esz;
      CUDA_OK(cudaMemcpy2DAsync(static_cast<char*>(dev) + (g.first_begin + p0) * esz, pitch,
                                static_cast<const char*>(host) + (row0 + g.first_begin + p0) * esz, pitch, width,
                                g.count, cudaMemcpyHostToDevice, c->copy_stream));
    };
    CUDA_OK(cudaEventRecord(c->ev[6], c->stream));  // buffers free of earlier users
    CUDA_OK(cudaStreamWaitEvent(c->copy_stream, c->ev[6], 0));
    for (uint32_t w = 0; w < n_win; ++w) {
      const uint64_t p0 = static_cast<uint64_t>(w) * win_rounds;
      for (const Group& g : groups) {
        if (g.len <= p0) continue;
        const uint64_t len = std::min<uint64_t>(win_rounds, g.len - p0);
        copy2d(c->pc.p, t->pc, 8, g, p0, len);
        copy2d(c->addr.p, t->data_addr, 8, g, p0, len);
        copy2d(c->op.p, t->op, 13, g, p0, len);
        copy2d(c->src.p, t->src, 16, g, p0, len);
        copy2d(c->dst.p, t->dst, 12, g, p0, len);
        copy2d(c->hist.p, t->hist, 28, g, p0, len);
        PackParams pp{};
        pp.n = g.count * len;
        pp.op = c->op.as<uint8_t>();
        pp.src = c->src.as<uint16_t>();
        pp.dst = c->dst.as<uint16_t>();
        pp.hist = c->hist.as<uint16_t>();
        pp.nc = c->nc_dev.as<NormConsts>();
        pp.stat = c->stat.as<float>();
        pp.iflags = c->iflags.as<uint8_t>();
        pp.seg_first = g.first_begin + p0;
        pp.seg_stride = g.stride;
        pp.seg_len = len;
        launch_pack(pp, c->copy_stream);
      }
      CUDA_OK(cudaEventRecord(c->win_ev[w], c->copy_stream));
    }
    CUDA_OK(cudaGetLastError());
  } else if (needs_input) {
    pack_if_needed(c, true);
  } else if (c->packed_gen == ~0ull || c->iflags.bytes < (P.g1 - P.g0)) {
    pack_if_needed(c, false);
  }
  uint32_t win_waited = 0;
  auto wait_windows = [&](uint32_t upto_round) {  // windows holding positions < upto_round
    while (win_waited < n_win && static_cast<uint64_t>(win_waited) * win_rounds < upto_round)
      CUDA_OK(cudaStreamWaitEvent(c->stream, c->win_ev[win_waited++], 0));
  };

  SubState* d_state = static_cast<SubState*>(c->state.need(K * sizeof(SubState)));
  CUDA_OK(cudaMemcpyAsync(d_state, hs.data(), K * sizeof(SubState), cudaMemcpyHostToDevice, c->stream));
  RingEntry* d_proc = static_cast<RingEntry*>(c->proc.need(K * pcap * sizeof(RingEntry)));
  RingEntry* d_wq = static_cast<RingEntry*>(c->wq.need(K * wcap * sizeof(RingEntry)));
  const uint64_t owned = P.own1 - P.own0;
  uint32_t* d_pf = cfg.record_fetch ? static_cast<uint32_t*>(c->pred_fetch.need(owned * 4)) : nullptr;

  // chunking of the batch (bounds activation memory; results are batch-independent)
  uint64_t chunk_cap = 65536;
  if (const char* e = std::getenv("SIMNET_CHUNK")) chunk_cap = std::max<long long>(8, std::atoll(e));  // tests
  const uint64_t chunk = std::min<uint64_t>(K, chunk_cap);
  // Fused round front (tensor-core C3): K1 apply + gather + conv chain in one
  // kernel, the gathered input stays in shared memory.  reserved[2] = 1 forces
  // the unfused path (ctx_kernel + TMA conv chain), e.g. for A/B checks.
  const bool fused = !oracle && c->model.tc != nullptr && tc_fused_front(c->model.tc) && cfg.reserved[2] == 0;
  if (!oracle && c->precision == ILSIM_PREC_FP8 && !fused)
    throw ApiError("fp8 precision runs only the fused rounds (C3 shape, reserved[2] = 0)");
  const bool capture_mode = c->cap_round != UINT32_MAX;
  const uint32_t dump_stride = input_stride(mc, ILSIM_PREC_FP32);  // fused capture: f32 rows of 100
  // gathered inputs: f32 rows of 100, or (bf16 inference) bf16 rows of 104
  const int xprec = oracle ? ILSIM_PREC_FP32 : c->precision;
  const uint32_t x_stride = needs_input ? input_stride(mc, xprec) : 0;
  const uint32_t x_floats = needs_input ? input_row_floats(mc) : 0;
  const bool x_split = !oracle && split_input(c->model);  // 3xTF32 hi/lo planes
  const uint64_t x_lo_off = x_split ? chunk * x_stride : 0;
  const uint64_t x_bytes = chunk * x_stride * input_elem_bytes(xprec) * (x_split ? 2 : 1);
  void* d_x = nullptr;
  if (fused) {
    if (capture_mode) d_x = c->x.need(chunk * dump_stride * sizeof(float));
  } else if (needs_input) {
    d_x = c->x.need(x_bytes);
    CUDA_OK(cudaMemsetAsync(d_x, 0, x_bytes, c->stream));  // bf16 row padding stays 0
  }
  ForwardBuffers fb{};
  if (!oracle) fb = forward_buffers(c->model, chunk, c->act, c->y);
  // fused rounds keep every chunk's FC1 partials until the next round's front
  // decodes them: partial planes for all K sub-traces, chunk f at part_off f
  if (fused && K > chunk) tc_prepare(c->model, K);
  auto fb_chunk = [&](uint64_t f) {
    ForwardBuffers b = fb;
    if (fused) b.part_off = f;
    return b;
  };

  // A "span" is a contiguous range [f, l) of sub-traces whose buffers start at
  // sample `off` of the chunk buffers, launched on stream `st`.
  auto x_at = [&](uint64_t off) -> void* {
    return d_x ? static_cast<void*>(static_cast<char*>(d_x) + off * x_stride * input_elem_bytes(xprec)) : nullptr;
  };
  auto make_ctx = [&](uint64_t f, uint64_t l, bool gather, uint64_t off) {
    CtxParams cp{};
    cp.state = d_state;
    cp.proc = d_proc;
    cp.wq = d_wq;
    cp.pmask = pcap - 1;
    cp.wmask = wcap - 1;
    cp.first = f;
    cp.last = l;
    cp.stat = c->stat.as<float>();
    cp.pc = c->pc.as<uint64_t>();
    cp.addr = c->addr.as<uint64_t>();
    cp.iflags = c->iflags.as<uint8_t>();
    cp.nc = c->nc_dev.as<NormConsts>();
    cp.x = x_at(off);
    cp.x_stride = x_stride;
    cp.x_floats = x_floats;
    cp.x_bf16 = xprec == ILSIM_PREC_BF16;
    cp.x_full = K > chunk;
    cp.x_split = x_split;
    cp.x_lo_off = x_lo_off;
    cp.max_context = mc;
    cp.bw = cfg.retire_bandwidth;
    cp.line = cfg.line_size;
    cp.page = cfg.page_size;
    cp.per_cycle = cfg.per_cycle_advance;
    cp.gather = gather && needs_input;
    return cp;
  };
  auto do_ctx = [&](uint64_t f, uint64_t l, bool gather, uint64_t off, cudaStream_t st) {
    const CtxParams cp = make_ctx(f, l, gather, off);
    launch_ctx(cp, st);
    return uint64_t{1};
  };
  auto decode_params = [&](uint64_t f, uint64_t l, const ForwardBuffers& fbs) {
    DecodeParams dp{};
    dp.state = d_state;
    dp.first = f;
    dp.last = l;
    dp.y = fbs.y;
    dp.y_stride = fbs.y_stride;
    dp.truth = oracle ? c->truth.as<uint32_t>() : nullptr;
    dp.iflags = c->iflags.as<uint8_t>();
    dp.nc = c->nc_dev.as<NormConsts>();
    dp.pred_fetch = d_pf;
    dp.class_fetch = c->cfg.class_fetch;
    dp.class_exec = c->cfg.class_exec;
    dp.class_store = c->cfg.class_store;
    dp.per_cycle = cfg.per_cycle_advance;
    return dp;
  };
  bool k3_fused = false;  // tensor-core tails run K3 themselves
  auto front_params = [&](uint64_t f, uint64_t l, float* dump, const ForwardBuffers& fbs) -> FrontParams {
    FrontParams fp{};
    fp.state = d_state;
    fp.proc = d_proc;
    fp.wq = d_wq;
    fp.pmask = pcap - 1;
    fp.wmask = wcap - 1;
    fp.first = f;
    fp.last = l;
    fp.stat = c->stat.as<float>();
    fp.stat_rows = c->g1 - c->g0;
    fp.pc = c->pc.as<uint64_t>();
    fp.addr = c->addr.as<uint64_t>();
    fp.iflags = c->iflags.as<uint8_t>();
    fp.nc = c->nc_dev.as<NormConsts>();
    fp.max_context = mc;
    fp.bw = cfg.retire_bandwidth;
    fp.line = cfg.line_size;
    fp.page = cfg.page_size;
    fp.per_cycle = cfg.per_cycle_advance;
    fp.dump = dump;
    fp.dump_stride = dump_stride;
    fp.fc = tc_fc_decode_args(c->model, l - f, fbs);
    fp.fc.pred_fetch = d_pf;
    fp.fc.per_cycle = cfg.per_cycle_advance;
    return fp;
  };
  // fused round: front (decode + apply of the previous round, gather, conv) -> FC1
  auto do_fc = [&](uint64_t f, uint64_t l, const ForwardBuffers& fbs, cudaStream_t st) -> uint64_t {
    k3_fused = true;
    return tc_fc(c->model, fbs.act[2], l - f, fbs, st, nullptr, false);
  };
  auto do_forward = [&](uint64_t f, uint64_t l, uint64_t off, const ForwardBuffers& fbs, cudaStream_t st) -> uint64_t {
    if (oracle) return 0;
    const DecodeParams dp = decode_params(f, l, fbs);
    return forward_launch(c->model, c->precision, x_at(off), x_stride, l - f, fbs, st, &dp, &k3_fused, x_lo_off);
  };
  auto do_decode = [&](uint64_t f, uint64_t l, const ForwardBuffers& fbs, cudaStream_t st) -> uint64_t {
    if (k3_fused) return 0;
    launch_decode(decode_params(f, l, fbs), st);
    return 1;
  };
  auto do_front = [&](uint64_t f, uint64_t l, float* dump, const ForwardBuffers& fbs, cudaStream_t st) -> uint64_t {
    return tc_front(c->model, front_params(f, l, dump, fbs), fbs, st);
  };
  // one round of one span: K1 -> K2 -> K3 (fused: front -> FC1)
  auto run_span = [&](uint64_t f, uint64_t l, uint64_t off, cudaStream_t st) -> uint64_t {
    ForwardBuffers fbs = oracle ? fb : fb_slice(c->model, fb, off);
    if (fused) fbs.part_off = f;
    if (fused) return do_front(f, l, nullptr, fbs, st) + do_fc(f, l, fbs, st);
    return do_ctx(f, l, true, off, st) + do_forward(f, l, off, fbs, st) + do_decode(f, l, fbs, st);
  };

  // rounds per CUDA graph: consecutive graph launches are not PDL-chained, so
  // longer graphs amortise that gap (SIMNET_GRAPH_ROUNDS overrides, tests / A/B)
  const uint32_t kGraphRounds = [] {
    const char* e = std::getenv("SIMNET_GRAPH_ROUNDS");
    const long v = e ? std::atol(e) : 16;
    return static_cast<uint32_t>(v >= 2 && v <= 1024 ? v : 16);
  }();
  auto launch_rounds = [&](uint32_t reps) -> uint64_t {
    uint64_t launches = 0;
    for (uint32_t r = 0; r < reps; ++r) {
      // SIMNET_CHAIN_TRACE: with a 16-round graph, only its middle round is
      // traced, so the buffer ends up holding a typical round (not the last)
      const bool traced_graph = rounds < kGraphRounds || reps == kGraphRounds;  // not the tail graph
      chain_trace_on() = traced_graph && (reps == 1 || r == reps / 2 || r == reps / 2 + 1);
      chain_trace_slot() = reps > 1 && r == reps / 2 + 1 ? 1 : 0;
      for (uint64_t f = 0; f < K; f += chunk) launches += run_span(f, std::min(K, f + chunk), 0, c->stream);
    }
    chain_trace_on() = true;
    chain_trace_slot() = 0;
    return launches;
  };

  // result collection (both the graph rounds and the persistent FC kernel)
  auto finish = [&](float ms, uint64_t launches, const double* kms) {
    CUDA_OK(cudaMemcpy(hs.data(), d_state, K * sizeof(SubState), cudaMemcpyDeviceToHost));
    if (predicted_fetch && d_pf)
      CUDA_OK(cudaMemcpy(predicted_fetch, d_pf, owned * 4, cudaMemcpyDeviceToHost));

    for (uint64_t j = 0; j < K; ++j) {
      const SubState& st = hs[j];
      const uint64_t i = P.sb + j;
      if (st.status == kErrStall)
        throw ApiError("processor queue stalled without progress at tick " + std::to_string(st.err_tick) +
                       " (sub-trace " + std::to_string(i) + ")");
      if (st.status == kErrDrain)
        throw ApiError("drain made no progress at tick " + std::to_string(st.err_tick) + " (sub-trace " +
                       std::to_string(i) + ")");
      if (st.status == kErrWriteRing)
        throw WriteRingOverflow("write queue ring overflow (capacity " + std::to_string(wcap) + ") in sub-trace " +
                                    std::to_string(i) + "; raise write_ring",
                                wcap);
      if (st.pos != st.len) throw ApiError("internal: sub-trace did not finish");
      ilsim_sub_result& r = subs[j];
      r.instructions = st.len - st.warm;
      r.total_cycles = st.cur - st.base_cur;
      r.sum_fetch = st.sum_fetch;
      r.delta = r.total_cycles - r.sum_fetch;
      r.drain_cycles = st.drain;
      r.overflow_stall_cycles = st.overflow - st.base_overflow;
      r.empty = r.instructions == 0;
      tot->total_cycles += r.total_cycles;
      tot->sum_fetch += r.sum_fetch;
      tot->delta += r.delta;
      tot->drain_cycles += r.drain_cycles;
      tot->overflow_stall_cycles += r.overflow_stall_cycles;
      tot->instructions += r.instructions;
    }
    tot->sub_traces = K;
    tot->rounds = rounds;
    tot->cpi = tot->instructions ? static_cast<double>(tot->total_cycles) / tot->instructions : 0.0;
    tot->device_ms = ms;
    for (int q = 0; q < 4; ++q) tot->kernel_ms[q] = kms[q];
    tot->launches = launches;
  };
  // Persistent kernels for the sequential configurations (seq_fc.cu): the
  // FC-only predictor at K <= 2 (c1) and the C3 at K = 1 (simulate_trace with
  // the CNN), fp32.  The whole simulation is one cooperative launch,
  // bit-identical to the launch-per-layer rounds below (SIMNET_NO_SEQ_FC=1
  // forces those, A/B; SIMNET_SEQ_TRACE=1 prints one round's phase times).
  {
    const ilsim_cnn_config& mcf = c->model.cfg;
    const ParamLayout& L = c->model.L;
    int dev = 0, ctas = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&ctas, cudaDevAttrMultiProcessorCount, dev));
    const bool eligible = !oracle && !capture_mode && cfg.reserved[0] == 0 && c->precision == ILSIM_PREC_FP32 &&
                          K == chunk && std::getenv("SIMNET_NO_SEQ_FC") == nullptr;
    const bool fc_seq = eligible && mcf.n_conv == 0 &&
                        seq_fc_fits(L.flat, mcf.fc_hidden, L.out_dim, static_cast<int>(K), ctas, static_cast<int>(pcap));
    const bool c3_shape = mcf.n_conv == 3 && mcf.conv[0] == 64 && mcf.conv[1] == 64 && mcf.conv[2] == 64 &&
                          mcf.input_channels == kSlots && mcf.sequence_length == 128 && !mcf.residual &&
                          L.flat == 1024 && mc + 1 <= 128;
    const bool c3_seq = eligible && c3_shape && K == 1 &&
                        seq_c3_fits(mcf.fc_hidden, L.out_dim, ctas, static_cast<int>(pcap));
    if (fc_seq || c3_seq) {
      // flags [0..3] (+ 16 trace words): zeroed before the launch
      const bool trace = std::getenv("SIMNET_SEQ_TRACE") != nullptr && rounds > 200;
      const size_t fbytes = 4 * sizeof(uint32_t) + (trace ? 16 * sizeof(long long) : 0);
      uint32_t* d_flags = static_cast<uint32_t*>(c->seq_flags.need(fbytes));
      long long* d_trace = trace ? reinterpret_cast<long long*>(d_flags + 4) : nullptr;
      CUDA_OK(cudaMemsetAsync(d_flags, 0, fbytes, c->stream));
      const float* P = c->model.params.as<float>();
      wait_windows(UINT32_MAX);
      CUDA_OK(cudaEventRecord(c->ev[0], c->stream));
      if (fc_seq) {
        SeqFcParams sp{};
        sp.ctx = make_ctx(0, K, true, 0);
        sp.dec = decode_params(0, K, fb);
        sp.w1 = P + L.fc1_w;
        sp.b1 = P + L.fc1_b;
        sp.w2 = P + L.fc2_w;
        sp.b2 = P + L.fc2_b;
        sp.flat = static_cast<int32_t>(L.flat);
        sp.hidden = mcf.fc_hidden;
        sp.od = L.out_dim;
        sp.h = fb.act[0];
        sp.y = fb.y;
        sp.flags = d_flags;
        sp.rounds = rounds;
        sp.trace = d_trace;
        launch_seq_fc(sp, ctas, c->stream);
      } else {
        SeqC3Params sp{};
        sp.ctx = make_ctx(0, K, true, 0);
        sp.dec = decode_params(0, K, fb);
        sp.w0 = P + L.w[0];
        sp.b0 = P + L.b[0];
        sp.w1c = P + L.w[1];
        sp.b1c = P + L.b[1];
        sp.w2c = P + L.w[2];
        sp.b2c = P + L.b[2];
        sp.w1f = P + L.fc1_w;
        sp.b1f = P + L.fc1_b;
        sp.w2f = P + L.fc2_w;
        sp.b2f = P + L.fc2_b;
        sp.hidden = mcf.fc_hidden;
        sp.od = L.out_dim;
        sp.flat = fb.act[2];
        sp.h = fb.act[3];
        sp.flags = d_flags;
        sp.rounds = rounds;
        sp.trace = d_trace;
        launch_seq_c3(sp, ctas, c->stream);
      }
      CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
      CUDA_OK(cudaGetLastError());
      CUDA_OK(cudaEventSynchronize(c->ev[1]));
      uint32_t hflags[4];
      CUDA_OK(cudaMemcpy(hflags, d_flags, sizeof(hflags), cudaMemcpyDeviceToHost));
      if (hflags[2] != 0) throw ApiError("persistent kernel: a CTA timed out waiting for its peers");
      if (trace) {  // diagnostics: phase boundaries of round 100 (ns); control words 0-7, worker 1 words 8-15
        long long tt[16];
        CUDA_OK(cudaMemcpy(tt, d_trace, sizeof(tt), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "%s round trace (ns), control:", fc_seq ? "seq_fc" : "seq_c3");
        for (int i = 1; i < 8; ++i)
          if (tt[i] != 0) std::fprintf(stderr, " %lld", tt[i] - tt[i - 1]);
        std::fprintf(stderr, " | worker 1:");
        for (int i = 9; i < 16; ++i)
          if (tt[i] != 0) std::fprintf(stderr, " %lld", tt[i] - tt[i - 1]);
        std::fprintf(stderr, "\n");
      }
      float ms = 0;
      CUDA_OK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
      const double zero[4] = {0, 0, 0, 0};
      finish(ms, 1, zero);
      return;
    }
  }
  if (capture_mode && K > chunk) throw ApiError("input capture needs a single chunk");
  if (capture_mode && !fused && xprec == ILSIM_PREC_BF16) throw ApiError("input capture needs f32 inputs");
  const bool profile = cfg.reserved[0] != 0;  // per-kernel event timing, no graphs
  // graphs: gN = kGraphRounds rounds (replayed), g1 = the remaining
  // rounds % kGraphRounds in one launch (graph boundaries are not PDL-chained)
  cudaGraphExec_t g1 = nullptr, gN = nullptr;
  uint64_t launches_1 = 0, launches_n = 0;
  const uint32_t tail_rounds = rounds % kGraphRounds;
  if (!capture_mode && !profile) {
    for (int which = 0; which < 2; ++which) {
      const uint32_t reps = which == 0 ? tail_rounds : kGraphRounds;
      if (reps == 0 || (which == 1 && rounds < kGraphRounds)) continue;
      cudaGraph_t g = nullptr;
      CUDA_OK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      try {
        (which == 0 ? launches_1 : launches_n) = launch_rounds(reps);
      } catch (...) {
        cudaStreamEndCapture(c->stream, &g);  // leave the stream usable
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        throw;
      }
      CUDA_OK(cudaStreamEndCapture(c->stream, &g));
      const cudaError_t ie = cudaGraphInstantiate(which == 0 ? &g1 : &gN, g, 0);
      cudaGraphDestroy(g);
      CUDA_OK(ie);
    }
  }

  CUDA_OK(cudaEventRecord(c->ev[0], c->stream));
  uint64_t launches = 0;
  double kms[4] = {0, 0, 0, 0};
  if (capture_mode || profile) {
    for (uint32_t r = 0; r < rounds; ++r) {
      for (uint64_t f = 0; f < K; f += chunk) {
        const uint64_t l = std::min(K, f + chunk);
        const bool cap_now = capture_mode && r == c->cap_round && needs_input;
        if (profile) CUDA_OK(cudaEventRecord(c->ev[2], c->stream));
        if (fused) {
          if (cap_now) CUDA_OK(cudaMemsetAsync(d_x, 0, chunk * dump_stride * sizeof(float), c->stream));
          launches += do_front(f, l, cap_now ? static_cast<float*>(d_x) : nullptr, fb_chunk(f), c->stream);
        } else {
          launches += do_ctx(f, l, true, 0, c->stream);
        }
        if (profile) CUDA_OK(cudaEventRecord(c->ev[3], c->stream));
        if (cap_now) {
          const uint32_t width = static_cast<uint32_t>(kSlots * (mc + 1));
          const uint64_t rows = std::min<uint64_t>(c->cap_rows, l - f);
          const uint32_t pitch = fused ? dump_stride : x_stride;
          CUDA_OK(cudaMemcpy2DAsync(c->cap_host, width * sizeof(float), d_x, pitch * sizeof(float),
                                    width * sizeof(float), rows, cudaMemcpyDeviceToHost, c->stream));
        }
        if (fused) {
          launches += do_fc(f, l, fb_chunk(f), c->stream);
        } else {
          launches += do_forward(f, l, 0, fb, c->stream);
        }
        if (profile) CUDA_OK(cudaEventRecord(c->ev[4], c->stream));
        launches += do_decode(f, l, fb, c->stream);
        if (profile) {
          CUDA_OK(cudaEventRecord(c->ev[5], c->stream));
          CUDA_OK(cudaEventSynchronize(c->ev[5]));
          float a = 0, b = 0, d = 0;
          CUDA_OK(cudaEventElapsedTime(&a, c->ev[2], c->ev[3]));
          CUDA_OK(cudaEventElapsedTime(&b, c->ev[3], c->ev[4]));
          CUDA_OK(cudaEventElapsedTime(&d, c->ev[4], c->ev[5]));
          kms[0] += a;
          kms[1] += b;
          kms[2] += d;
        }
      }
    }
  } else {
    uint32_t r = 0;
    while (gN && r + kGraphRounds <= rounds) {
      wait_windows(r + kGraphRounds);
      CUDA_OK(cudaGraphLaunch(gN, c->stream));
      launches += launches_n;
      r += kGraphRounds;
    }
    if (r < rounds) {  // the tail, one launch
      wait_windows(rounds);
      CUDA_OK(cudaGraphLaunch(g1, c->stream));
      launches += launches_1;
      r = rounds;
    }
  }
  wait_windows(UINT32_MAX);
  for (uint64_t f = 0; f < K; f += chunk) {  // apply final step, drain
    const uint64_t l = std::min(K, f + chunk);
    if (fused) {
      launch_final_decode(front_params(f, l, nullptr, fb_chunk(f)), c->stream);
      ++launches;
    } else {
      launches += do_ctx(f, l, false, 0, c->stream);
    }
  }
  CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaEventSynchronize(c->ev[1]));
  if (g1) cudaGraphExecDestroy(g1);
  if (gN) cudaGraphExecDestroy(gN);
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));

  finish(ms, launches, kms);
}

// run_impl, rerun with a doubled write ring while a sub-trace's write queue
// outgrows it and the caller left write_ring on auto (0); the reference's write
// queue is an unbounded deque (simcore.hpp:61-90).  Bounded at 2^22 entries
// and 64 GB of rings; past that the overflow is reported.
template <class Reset>
void run_growing_ring(ilsim_gpu_ctx* c, const ilsim_sim_config& cfg, ilsim_sub_result* subs, uint64_t sub_cap,
                      uint32_t* predicted_fetch, ilsim_totals* totals, Reset reset) {
  ilsim_sim_config cur = cfg;
  for (;;) {
    try {
      *totals = ilsim_totals{};
      run_impl(c, cur, subs, sub_cap, predicted_fetch, totals);
      return;
    } catch (const WriteRingOverflow& e) {
      const uint64_t next = 2ull * e.capacity;
      const uint64_t k = cur.shard_end > cur.shard_begin ? cur.shard_end - cur.shard_begin : std::max<uint64_t>(cur.k, 1);
      if (cfg.write_ring != 0 || next > (1ull << 22) || next * k * sizeof(RingEntry) > (64ull << 30)) throw;
      cur.write_ring = static_cast<int32_t>(next);
      reset();
    }
  }
}

// Shared tail of the trace loaders: flags + (model loaded) normalised static
// slots of the uploaded slice, then the trace is ready.
void finish_trace_load(ilsim_gpu_ctx* c, uint64_t m) {
  c->packed_gen = ~0ull;
  c->iflags.need(m);
  // static slots depend on the model's NormStats: pack now if a model is loaded
  if (m) {
    PackParams pp{};
    pp.n = m;
    pp.op = c->op.as<uint8_t>();
    pp.src = c->src.as<uint16_t>();
    pp.dst = c->dst.as<uint16_t>();
    pp.hist = c->hist.as<uint16_t>();
    pp.nc = c->nc_dev.as<NormConsts>();
    pp.stat = c->has_model ? static_cast<float*>(c->stat.need(m * kStatStride * sizeof(float))) : nullptr;
    pp.iflags = c->iflags.as<uint8_t>();
    launch_pack(pp, c->stream);
    CUDA_OK(cudaGetLastError());
    if (c->has_model) c->packed_gen = c->model_gen;
  }
  CUDA_OK(cudaStreamSynchronize(c->stream));
  c->has_trace = true;
}

}  // namespace

// --------------------------------------------------------------------------
// C-ABI
// --------------------------------------------------------------------------
namespace {
void put_err(char* err, int n, const std::string& m) {
  if (err && n > 0) {
    std::strncpy(err, m.c_str(), static_cast<size_t>(n) - 1);
    err[n - 1] = 0;
  }
}

template <typename F>
int guard(ilsim_gpu_ctx* c, F&& f) {
  try {
    if (c) CUDA_OK(cudaSetDevice(c->device));
    f();
    if (c) c->err.clear();
    return 0;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

// Diagnostics only (not in ilsim_gpu.h): copy the conv-chain event clocks of
// the last traced launch (SIMNET_CHAIN_TRACE=1) into out[148*32].
int simnet_debug_chain_trace(long long* out) {
  long long* p = chain_trace_ptr();
  if (!p) return 1;
  return cudaMemcpy(out, p, 148 * 32 * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
}

// Diagnostics only: copy n words of the trace buffer (front + FC1 event clocks).
int simnet_debug_chain_trace_full(long long* out, int n) {
  long long* p = chain_trace_ptr();
  if (!p) return 1;
  return cudaMemcpy(out, p, static_cast<size_t>(n) * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
}

int ilsim_gpu_abi_version(void) { return ILSIM_GPU_ABI_VERSION; }

int ilsim_gpu_create(const ilsim_gpu_options* o, ilsim_gpu_ctx** out, char* err, int errlen) {
  try {
    auto c = std::make_unique<ilsim_gpu_ctx>();
    c->device = o ? o->device : 0;
    c->precision = o ? o->precision : ILSIM_PREC_FP32;
    if (c->precision < ILSIM_PREC_FP32 || c->precision > ILSIM_PREC_FP8)
      throw ApiError("unknown precision");
    int count = 0;
    CUDA_OK(cudaGetDeviceCount(&count));
    if (c->device < 0 || c->device >= count) throw ApiError("CUDA device out of range");
    CUDA_OK(cudaSetDevice(c->device));
    cudaDeviceProp prop{};
    CUDA_OK(cudaGetDeviceProperties(&prop, c->device));
    if (prop.major != 10) throw ApiError("this build targets sm_100a (B200); found sm_" +
                                         std::to_string(prop.major) + std::to_string(prop.minor));
    CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    for (auto& e : c->ev) CUDA_OK(cudaEventCreate(&e));
    set_norm(c.get(), nullptr);
    *out = c.release();
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

void ilsim_gpu_destroy(ilsim_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->win_ev) cudaEventDestroy(e);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* ilsim_gpu_last_error(const ilsim_gpu_ctx* c) { return c ? c->err.c_str() : ""; }

int ilsim_gpu_load_model(ilsim_gpu_ctx* c, const ilsim_cnn_config* cfg, const double* norm,
                         const float* params, uint64_t n_params) {
  return guard(c, [&] {
    validate_config(*cfg);
    if (n_params != param_count_of(*cfg)) throw ApiError("model parameter count mismatch");
    c->cfg = *cfg;
    c->norm.assign(norm, norm + 106);
    set_norm(c, norm);
    model_upload(c->model, *cfg, params, c->precision, c->stream);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->has_model = true;
    ++c->model_gen;
  });
}

int ilsim_gpu_load_trace(ilsim_gpu_ctx* c, const ilsim_trace_view* t, const ilsim_sim_config* cfg) {
  return guard(c, [&] {
    const Plan P = make_plan(*cfg, t->n);
    c->has_trace = false;
    c->t_total = t->n;
    c->g0 = P.g0;
    c->g1 = P.g1;
    const uint64_t g0 = view_row(t, P), m = P.g1 - P.g0;
    upload(c->pc, t->pc + g0, m, c->stream);
    upload(c->addr, t->data_addr + g0, m, c->stream);
    upload(c->op, t->op + 13 * g0, 13 * m, c->stream);
    upload(c->src, t->src + 8 * g0, 8 * m, c->stream);
    upload(c->dst, t->dst + 6 * g0, 6 * m, c->stream);
    upload(c->hist, t->hist + 14 * g0, 14 * m, c->stream);
    c->has_truth = t->truth != nullptr;
    if (c->has_truth) upload(c->truth, t->truth + 3 * g0, 3 * m, c->stream);
    finish_trace_load(c, m);
  });
}

int ilsim_gpu_load_trace_records(ilsim_gpu_ctx* c, const void* records, uint64_t n, const ilsim_sim_config* cfg,
                                 int32_t with_truth) {
  return guard(c, [&] {
    const Plan P = make_plan(*cfg, n);
    c->has_trace = false;
    c->t_total = n;
    c->g0 = P.g0;
    c->g1 = P.g1;
    const uint64_t g0 = P.g0, m = P.g1 - P.g0;
    constexpr uint64_t kRec = 108, kStageRecs = 1ull << 22;  // 432 MB staging at most
    c->pc.need(m * 8);
    c->addr.need(m * 8);
    c->op.need(m * 13);
    c->src.need(m * 16);
    c->dst.need(m * 12);
    c->hist.need(m * 28);
    c->has_truth = with_truth != 0;
    if (c->has_truth) c->truth.need(m * 12);
    if (m) {
      void* stage = c->rec_stage.need(std::min(m, kStageRecs) * kRec);
      const uint8_t* src = static_cast<const uint8_t*>(records) + g0 * kRec;
      for (uint64_t f = 0; f < m; f += kStageRecs) {
        const uint64_t k = std::min(kStageRecs, m - f);
        CUDA_OK(cudaMemcpyAsync(stage, src + f * kRec, k * kRec, cudaMemcpyHostToDevice, c->stream));
        UnpackParams u{};
        u.rec = static_cast<const uint8_t*>(stage);
        u.n = k;
        u.pc = c->pc.as<uint64_t>() + f;
        u.addr = c->addr.as<uint64_t>() + f;
        u.op = c->op.as<uint8_t>() + 13 * f;
        u.src = c->src.as<uint16_t>() + 8 * f;
        u.dst = c->dst.as<uint16_t>() + 6 * f;
        u.hist = c->hist.as<uint16_t>() + 14 * f;
        u.truth = c->has_truth ? c->truth.as<uint32_t>() + 3 * f : nullptr;
        launch_unpack_records(u, c->stream);
        CUDA_OK(cudaGetLastError());
      }
    }
    finish_trace_load(c, m);
  });
}

int ilsim_gpu_run(ilsim_gpu_ctx* c, const ilsim_sim_config* cfg, ilsim_sub_result* subs, uint64_t sub_cap,
                  uint32_t* predicted_fetch, ilsim_totals* totals) {
  return guard(c, [&] { run_growing_ring(c, *cfg, subs, sub_cap, predicted_fetch, totals, [] {}); });
}

int ilsim_gpu_simulate_parallel(ilsim_gpu_ctx* c, const ilsim_trace_view* t, const ilsim_sim_config* cfg,
                                ilsim_sub_result* subs, uint64_t sub_cap, uint32_t* predicted_fetch,
                                ilsim_totals* totals) {
  // Large model-driven runs upload the trace window by window, overlapped
  // with the rounds (one call borrows the view for its whole duration).
  // (truth latencies, if present in the view, are not needed by a model-driven run)
  const bool overlap = c && t && cfg && c->has_model && cfg->oracle == 0 &&
                       cfg->reserved[0] == 0 && cfg->reserved[1] == 0 && c->cap_round == UINT32_MAX &&
                       t->n >= (1ull << 20) &&
                       !std::getenv("SIMNET_NO_UPLOAD_OVERLAP");
  if (!overlap) {
    if (ilsim_gpu_load_trace(c, t, cfg) != 0) return 1;
    return ilsim_gpu_run(c, cfg, subs, sub_cap, predicted_fetch, totals);
  }
  const int rc = guard(c, [&] {
    const Plan P = make_plan(*cfg, t->n);
    view_row(t, P);
    c->has_trace = false;
    c->t_total = t->n;
    c->g0 = P.g0;
    c->g1 = P.g1;
    const uint64_t m = P.g1 - P.g0;
    c->pc.need(m * 8);
    c->addr.need(m * 8);
    c->op.need(m * 13);
    c->src.need(m * 16);
    c->dst.need(m * 12);
    c->hist.need(m * 28);
    c->has_truth = false;
    c->iflags.need(m);
    c->stat.need(m * kStatStride * sizeof(float));
    c->packed_gen = c->model_gen;  // packed window by window in run_impl
    c->has_trace = true;
    if (!c->copy_stream) CUDA_OK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    c->deferred = t;
    try {
      // a rerun with a larger write ring uploads and packs the windows again
      run_growing_ring(c, *cfg, subs, sub_cap, predicted_fetch, totals, [&] {
        c->packed_gen = c->model_gen;
        c->has_trace = true;
      });
    } catch (...) {
      c->deferred = nullptr;
      c->packed_gen = ~0ull;  // the device trace may be partial: it must be loaded again
      c->has_trace = false;
      cudaStreamSynchronize(c->copy_stream);
      throw;
    }
    c->deferred = nullptr;
  });
  return rc;
}

int ilsim_gpu_predict(ilsim_gpu_ctx* c, const float* inputs, uint64_t n, const uint8_t* is_store,
                      float* outputs, uint32_t* triples) {
  return guard(c, [&] {
    if (!c->has_model) throw ApiError("no model loaded");
    if (n == 0) return;
    const int mc = c->cfg.max_context;
    const uint32_t width = static_cast<uint32_t>(kSlots * (mc + 1));
    const uint32_t x_stride = input_stride(mc, c->precision);
    const uint64_t chunk = std::min<uint64_t>(n, 65536);
    const uint64_t x_lo_off = split_input(c->model) ? chunk * x_stride : 0;
    const uint64_t x_bytes = chunk * x_stride * input_elem_bytes(c->precision) * (x_lo_off ? 2 : 1);
    void* d_x = c->x.need(x_bytes);
    ForwardBuffers fb = forward_buffers(c->model, chunk, c->act, c->y);
    DevBuf d_store, d_trip, d_in;
    uint8_t* ds = static_cast<uint8_t*>(d_store.need(chunk));
    uint32_t* dt = static_cast<uint32_t*>(d_trip.need(chunk * 12));
    float* din = static_cast<float*>(d_in.need(chunk * width * sizeof(float)));
    for (uint64_t f = 0; f < n; f += chunk) {
      const uint64_t m = std::min(chunk, n - f);
      CUDA_OK(cudaMemsetAsync(d_x, 0, x_bytes, c->stream));
      CUDA_OK(cudaMemcpyAsync(din, inputs + f * width, m * width * sizeof(float), cudaMemcpyHostToDevice,
                              c->stream));
      launch_pack_inputs(din, m, width, d_x, x_stride, c->precision == ILSIM_PREC_BF16, x_lo_off, c->stream);
      CUDA_OK(cudaMemcpyAsync(ds, is_store + f, m, cudaMemcpyHostToDevice, c->stream));
      forward_launch(c->model, c->precision, d_x, x_stride, m, fb, c->stream, nullptr, nullptr, x_lo_off);
      launch_decode_only(fb.y, fb.y_stride, m, ds, c->nc_dev.as<NormConsts>(), c->cfg.class_fetch,
                         c->cfg.class_exec, c->cfg.class_store, dt, c->stream);
      CUDA_OK(cudaGetLastError());
      const int od = output_dim_of(c->cfg);
      if (outputs)
        CUDA_OK(cudaMemcpy2DAsync(outputs + f * od, od * sizeof(float), fb.y, fb.y_stride * sizeof(float),
                                  od * sizeof(float), m, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OK(cudaMemcpyAsync(triples + 3 * f, dt, m * 12, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OK(cudaStreamSynchronize(c->stream));
    }
  });
}

int ilsim_gpu_decode_outputs(ilsim_gpu_ctx* c, const float* outputs, uint64_t n, const uint8_t* is_store,
                             uint32_t* triples, int32_t path) {
  return guard(c, [&] {
    if (!c->has_model) throw ApiError("no model loaded");
    if (path != 0 && path != 1) throw ApiError("decode path must be 0 (per-thread) or 1 (warp)");
    if (n == 0) return;
    const int od = output_dim_of(c->cfg);
    DevBuf d_y, d_store, d_trip;
    float* dy = static_cast<float*>(d_y.need(n * od * sizeof(float)));
    uint8_t* ds = static_cast<uint8_t*>(d_store.need(n));
    uint32_t* dt = static_cast<uint32_t*>(d_trip.need(n * 12));
    CUDA_OK(cudaMemcpyAsync(dy, outputs, n * od * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(ds, is_store, n, cudaMemcpyHostToDevice, c->stream));
    (path == 0 ? launch_decode_only : launch_decode_warp)(dy, od, n, ds, c->nc_dev.as<NormConsts>(),
                                                           c->cfg.class_fetch, c->cfg.class_exec,
                                                           c->cfg.class_store, dt, c->stream);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpyAsync(triples, dt, n * 12, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int ilsim_gpu_set_capture(ilsim_gpu_ctx* c, uint32_t round, float* inputs, uint64_t rows) {
  return guard(c, [&] {
    c->cap_round = round;
    c->cap_host = inputs;
    c->cap_rows = rows;
  });
}

int ilsim_gpu_partition(uint64_t n, uint64_t k, uint64_t* starts, char* err, int errlen) {
  try {
    const auto s = partition_starts(n, k);
    std::copy(s.begin(), s.end(), starts);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

uint64_t ilsim_gpu_model_flops(const ilsim_cnn_config* cfg) { return model_flops_of(*cfg); }
uint64_t ilsim_gpu_param_count(const ilsim_cnn_config* cfg) { return param_count_of(*cfg); }

int ilsim_gpu_init_weights(const ilsim_cnn_config* cfg, uint64_t seed, float* params, uint64_t n, char* err,
                           int errlen) {
  try {
    validate_config(*cfg);
    if (n != param_count_of(*cfg)) throw ApiError("parameter buffer size mismatch");
    init_weights_into(*cfg, seed, params);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Multi-device group: the C++ drop-in for simulate_parallel over several GPUs
// of one process (parallel.cpp:26-93 with the sub-traces sharded contiguously,
// SURVEY.md §8(e)).  One context and one host thread per device; each thread
// uploads only its shard's slice of the borrowed trace view and runs its
// rounds; the per-sub-trace results land in the caller's arrays in sub-trace
// order and the totals are summed on the host exactly as parallel.cpp:83-92
// sums sub_results (integer sums: identical for any device count).
// ---------------------------------------------------------------------------
struct ilsim_gpu_group {
  std::vector<ilsim_gpu_ctx*> ctx;
  std::string err;
};

extern "C" {

int ilsim_gpu_group_create(const ilsim_gpu_options* opts, const int32_t* devices, int32_t n_devices,
                           ilsim_gpu_group** out, char* err, int errlen) {
  try {
    if (!out) throw ApiError("null output pointer");
    if (n_devices < 1 || !devices) throw ApiError("a device group needs at least one device");
    auto g = std::make_unique<ilsim_gpu_group>();
    for (int32_t i = 0; i < n_devices; ++i) {
      ilsim_gpu_options o = opts ? *opts : ilsim_gpu_options{};
      o.device = devices[i];
      ilsim_gpu_ctx* c = nullptr;
      char e[512] = {0};
      if (ilsim_gpu_create(&o, &c, e, sizeof(e)) != 0) {
        for (auto* x : g->ctx) ilsim_gpu_destroy(x);
        throw ApiError("device " + std::to_string(devices[i]) + ": " + e);
      }
      g->ctx.push_back(c);
    }
    *out = g.release();
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

void ilsim_gpu_group_destroy(ilsim_gpu_group* g) {
  if (!g) return;
  for (auto* c : g->ctx) ilsim_gpu_destroy(c);
  delete g;
}

const char* ilsim_gpu_group_last_error(const ilsim_gpu_group* g) { return g ? g->err.c_str() : ""; }

int ilsim_gpu_group_size(const ilsim_gpu_group* g) { return g ? static_cast<int>(g->ctx.size()) : 0; }

int ilsim_gpu_group_load_model(ilsim_gpu_group* g, const ilsim_cnn_config* cfg, const double* norm,
                               const float* params, uint64_t n_params) {
  if (!g) return 1;
  for (size_t i = 0; i < g->ctx.size(); ++i)
    if (ilsim_gpu_load_model(g->ctx[i], cfg, norm, params, n_params) != 0) {
      g->err = "device " + std::to_string(g->ctx[i]->device) + ": " + g->ctx[i]->err;
      return 1;
    }
  g->err.clear();
  return 0;
}

int ilsim_gpu_group_simulate_parallel(ilsim_gpu_group* g, const ilsim_trace_view* t, const ilsim_sim_config* cfg,
                                      ilsim_sub_result* subs, uint64_t sub_cap, uint32_t* predicted_fetch,
                                      ilsim_totals* totals) {
  if (!g) return 1;
  try {
    if (!t || !cfg || !totals) throw ApiError("null argument");
    if (cfg->shard_begin != 0 || cfg->shard_end != 0)
      throw ApiError("a device group shards the partition itself (shard_begin / shard_end must be 0)");
    *totals = ilsim_totals{};
    const size_t nd = g->ctx.size();
    // the global partition (validation errors with the reference's texts)
    const Plan P = make_plan(*cfg, t->n);
    const uint64_t k = cfg->sequential ? 1 : P.k;
    if (t->n == 0 || cfg->sequential || nd == 1) {  // one device does it all (simcore.cpp:185-196)
      if (ilsim_gpu_simulate_parallel(g->ctx[0], t, cfg, subs, sub_cap, predicted_fetch, totals) != 0)
        throw ApiError(g->ctx[0]->err);
      g->err.clear();
      return 0;
    }
    if (k > sub_cap) throw ApiError("sub_cap too small");
    std::vector<ilsim_totals> tot(nd);
    std::vector<std::string> errs(nd);
    std::vector<std::thread> th;
    for (size_t d = 0; d < nd; ++d) {
      // contiguous blocks, the first k % nd devices one sub-trace more (dist.shard_range)
      const uint64_t base = k / nd, rem = k % nd;
      const uint64_t sb = d * base + std::min<uint64_t>(d, rem);
      const uint64_t se = sb + base + (d < rem ? 1 : 0);
      if (sb == se) continue;
      th.emplace_back([&, d, sb, se] {
        ilsim_sim_config c = *cfg;
        c.shard_begin = sb;
        c.shard_end = se;
        const uint64_t own0 = P.starts[sb];
        if (ilsim_gpu_simulate_parallel(g->ctx[d], t, &c, subs + sb, se - sb,
                                        predicted_fetch ? predicted_fetch + own0 : nullptr, &tot[d]) != 0)
          errs[d] = "device " + std::to_string(g->ctx[d]->device) + ": " + g->ctx[d]->err;
      });
    }
    for (auto& x : th) x.join();
    for (const auto& e : errs)
      if (!e.empty()) throw ApiError(e);
    for (const auto& x : tot) {
      totals->sub_traces += x.sub_traces;
      totals->instructions += x.instructions;
      totals->total_cycles += x.total_cycles;
      totals->sum_fetch += x.sum_fetch;
      totals->delta += x.delta;
      totals->drain_cycles += x.drain_cycles;
      totals->overflow_stall_cycles += x.overflow_stall_cycles;
      totals->rounds = std::max(totals->rounds, x.rounds);
      totals->device_ms = std::max(totals->device_ms, x.device_ms);  // the slowest device
      for (int q = 0; q < 4; ++q) totals->kernel_ms[q] = std::max(totals->kernel_ms[q], x.kernel_ms[q]);
      totals->launches += x.launches;
    }
    totals->cpi = totals->instructions ? static_cast<double>(totals->total_cycles) / totals->instructions : 0.0;
    g->err.clear();
    return 0;
  } catch (const std::exception& e) {
    g->err = e.what();
    return 1;
  }
}

}  // extern "C"
