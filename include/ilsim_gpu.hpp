// ilsim_gpu.hpp — header-only C++ adapter from the reference's types
// (ilsim::AnnotatedInstruction, ModelWeights, ParallelConfig, ParallelResult;
// /root/reference/proj/include/ilsim) onto the C-ABI in ilsim_gpu.h.
//
// A reference maintainer adds this next to parallel.hpp and calls
//   ilsim::gpu::simulate_parallel_gpu(trace, weights, config)
// wherever simulate_parallel(trace, cnn_predictor, config) is called today
// (tools/ilsim_main.cpp:148-169, bindings/module.cpp:131-155).  Errors are
// rethrown as ilsim::Error with the library's message.
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "ilsim/cnn.hpp"
#include "ilsim/parallel.hpp"
#include "ilsim/predictor.hpp"
#include "ilsim_gpu.h"

namespace ilsim::gpu {

namespace detail {

struct Soa {  // AnnotatedInstruction (trace.hpp:98-109) -> structure of arrays
  std::vector<uint64_t> pc, addr;
  std::vector<uint8_t> op, has;
  std::vector<uint16_t> src, dst, hist;
  std::vector<uint32_t> truth;
  ilsim_trace_view view{};
  explicit Soa(std::span<const AnnotatedInstruction> t) {
    const size_t n = t.size();
    pc.resize(n);
    addr.resize(n);
    has.resize(n);
    op.resize(n * 13);
    src.resize(n * 8);
    dst.resize(n * 6);
    hist.resize(n * 14);
    truth.resize(n * 3);
    for (size_t i = 0; i < n; ++i) {
      const auto& a = t[i];
      pc[i] = a.stat.pc;
      addr[i] = a.stat.has_data ? a.stat.data_addr : 0;
      has[i] = a.stat.has_data ? 1 : 0;
      for (int j = 0; j < 13; ++j) op[i * 13 + j] = a.stat.op[j];
      for (int j = 0; j < 8; ++j) src[i * 8 + j] = a.stat.src[j];
      for (int j = 0; j < 6; ++j) dst[i * 6 + j] = a.stat.dst[j];
      for (int j = 0; j < 14; ++j) hist[i * 14 + j] = a.hist.v[j];
      truth[i * 3 + 0] = a.truth.fetch;
      truth[i * 3 + 1] = a.truth.execution;
      truth[i * 3 + 2] = a.truth.store;
    }
    view = ilsim_trace_view{n, pc.data(), op.data(), src.data(), dst.data(), has.data(), addr.data(), hist.data(),
                            truth.data(), 0};
  }
};


inline ilsim_sim_config sim_config(const ParallelConfig& pc, bool oracle) {
  ilsim_sim_config c{};
  c.k = pc.k;
  c.subtrace_size = pc.subtrace_size;
  c.batch_max = pc.batch_max;
  c.max_context = pc.sim.max_context;
  c.retire_bandwidth = pc.sim.retire_bandwidth;
  c.per_cycle_advance = pc.sim.per_cycle_advance ? 1 : 0;
  c.record_fetch = pc.sim.record_fetch ? 1 : 0;
  c.oracle = oracle ? 1 : 0;
  c.line_size = pc.sim.line_size;
  c.page_size = pc.sim.page_size;
  return c;
}

inline uint64_t sub_count(size_t n, const ParallelConfig& pc) {
  uint64_t k = pc.k;
  if (pc.subtrace_size > 0 && k == 0) k = n == 0 ? 1 : (n + pc.subtrace_size - 1) / pc.subtrace_size;
  return k == 0 ? 1 : k;
}

// C-ABI outputs -> ParallelResult (parallel.hpp:31-38)
inline ParallelResult to_result(size_t n, const std::vector<ilsim_sub_result>& subs, const ilsim_totals& tot,
                                std::vector<uint32_t>&& fetch) {
  ParallelResult out;
  out.instructions = n;
  size_t off = 0;
  for (uint64_t i = 0; i < tot.sub_traces; ++i) {
    SimResult r;
    r.instructions = subs[i].instructions;
    r.total_cycles = subs[i].total_cycles;
    r.sum_fetch = subs[i].sum_fetch;
    r.delta = subs[i].delta;
    r.drain_cycles = subs[i].drain_cycles;
    r.overflow_stall_cycles = subs[i].overflow_stall_cycles;
    r.empty = subs[i].empty != 0;
    r.cpi = r.instructions ? static_cast<double>(r.total_cycles) / r.instructions : 0.0;
    if (!fetch.empty()) r.predicted_fetch.assign(fetch.begin() + off, fetch.begin() + off + r.instructions);
    off += r.instructions;
    out.total_cycles += r.total_cycles;
    out.sub_results.push_back(std::move(r));
  }
  out.cpi = n == 0 ? 0.0 : static_cast<double>(out.total_cycles) / n;
  out.predicted_fetch = std::move(fetch);
  return out;
}

// load_model (cnn.cpp:662-697) output -> the C-ABI's config + NormStats
inline ilsim_cnn_config cnn_config(const ModelWeights& w, double* norm) {
  ilsim_cnn_config c{};
  c.input_channels = w.config.input_channels;
  c.max_context = w.config.max_context;
  c.sequence_length = w.config.sequence_length;
  c.n_conv = static_cast<int32_t>(w.config.conv_channels.size());
  for (int i = 0; i < c.n_conv && i < 8; ++i) c.conv[i] = w.config.conv_channels[i];
  c.fc_hidden = w.config.fc_hidden;
  c.class_fetch = w.config.class_fetch;
  c.class_exec = w.config.class_exec;
  c.class_store = w.config.class_store;
  c.residual = w.config.residual_blocks ? 1 : 0;
  for (int k = 0; k < 50; ++k) {
    norm[k] = w.norm.mean[k];
    norm[50 + k] = w.norm.stdev[k];
  }
  for (int k = 0; k < 3; ++k) {
    norm[100 + k] = w.norm.label_mean[k];
    norm[103 + k] = w.norm.label_stdev[k];
  }
  return c;
}

}  // namespace detail

class Context {
public:
  explicit Context(int device = 0, int precision = ILSIM_PREC_TF32X3) {
    ilsim_gpu_options o{};
    o.device = device;
    o.precision = precision;
    char err[512] = {0};
    if (ilsim_gpu_create(&o, &ctx_, err, sizeof err) != 0) throw Error(err);
  }
  ~Context() { ilsim_gpu_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  // load_model (cnn.cpp:662-697) output -> device (CnnPredictor ctor).
  void load_model(const ModelWeights& w) {
    double norm[106];
    const ilsim_cnn_config c = detail::cnn_config(w, norm);
    check(ilsim_gpu_load_model(ctx_, &c, norm, w.params.data(), w.params.size()));
    max_context_ = w.config.max_context;
  }

  // simulate_parallel (parallel.cpp:26-93) on the GPU.
  ParallelResult simulate_parallel(std::span<const AnnotatedInstruction> trace, const ParallelConfig& pc,
                                   bool oracle = false) {
    detail::Soa soa(trace);
    const ilsim_sim_config c = detail::sim_config(pc, oracle);
    std::vector<ilsim_sub_result> subs(detail::sub_count(trace.size(), pc));
    std::vector<uint32_t> fetch(pc.sim.record_fetch ? trace.size() : 0);
    ilsim_totals tot{};
    check(ilsim_gpu_simulate_parallel(ctx_, &soa.view, &c, subs.data(), subs.size(),
                                      fetch.empty() ? nullptr : fetch.data(), &tot));
    return detail::to_result(trace.size(), subs, tot, std::move(fetch));
  }

  // CnnPredictor::predict (predictor.cpp:13-29) on the GPU: inference + hybrid
  // decode of the requests' inputs (PredictRequest::input layout).
  void predict(std::span<const PredictRequest> requests, std::span<LatencyTriple> out) {
    if (out.size() != requests.size()) throw Error("predict: output span size differs from the requests");
    const size_t width = static_cast<size_t>(FeatureLayout::kSlots) * static_cast<size_t>(max_context_ + 1);
    std::vector<float> in(requests.size() * width);
    std::vector<uint8_t> st(requests.size());
    for (size_t i = 0; i < requests.size(); ++i) {
      std::copy(requests[i].input, requests[i].input + width, in.begin() + static_cast<std::ptrdiff_t>(i * width));
      st[i] = requests[i].target_is_store ? 1 : 0;
    }
    std::vector<uint32_t> tri(requests.size() * 3);
    if (!requests.empty()) check(ilsim_gpu_predict(ctx_, in.data(), requests.size(), st.data(), nullptr, tri.data()));
    for (size_t i = 0; i < requests.size(); ++i) out[i] = LatencyTriple{tri[3 * i], tri[3 * i + 1], tri[3 * i + 2]};
  }

private:
  void check(int rc) {
    if (rc != 0) throw Error(ilsim_gpu_last_error(ctx_));
  }

  ilsim_gpu_ctx* ctx_ = nullptr;
  int max_context_ = 110;
};

// Drop-in for `simulate_parallel(trace, CnnPredictor(weights), config)`.
inline ParallelResult simulate_parallel_gpu(std::span<const AnnotatedInstruction> trace, const ModelWeights& w,
                                            const ParallelConfig& config, int device = 0,
                                            int precision = ILSIM_PREC_TF32X3) {
  Context ctx(device, precision);
  ctx.load_model(w);
  return ctx.simulate_parallel(trace, config);
}

// Several GPUs of one process behind one simulate_parallel
// (ilsim_gpu_group_*: one host thread per device inside the library).
class Group {
public:
  explicit Group(const std::vector<int>& devices, int precision = ILSIM_PREC_TF32X3) {
    ilsim_gpu_options o{};
    o.precision = precision;
    std::vector<int32_t> d(devices.begin(), devices.end());
    char err[512] = {0};
    if (ilsim_gpu_group_create(&o, d.data(), static_cast<int32_t>(d.size()), &g_, err, sizeof err) != 0)
      throw Error(err);
  }
  ~Group() { ilsim_gpu_group_destroy(g_); }
  Group(const Group&) = delete;
  Group& operator=(const Group&) = delete;

  void load_model(const ModelWeights& w) {
    double norm[106];
    const ilsim_cnn_config c = detail::cnn_config(w, norm);
    check(ilsim_gpu_group_load_model(g_, &c, norm, w.params.data(), w.params.size()));
  }

  ParallelResult simulate_parallel(std::span<const AnnotatedInstruction> trace, const ParallelConfig& pc,
                                   bool oracle = false) {
    detail::Soa soa(trace);
    const ilsim_sim_config c = detail::sim_config(pc, oracle);
    std::vector<ilsim_sub_result> subs(detail::sub_count(trace.size(), pc));
    std::vector<uint32_t> fetch(pc.sim.record_fetch ? trace.size() : 0);
    ilsim_totals tot{};
    check(ilsim_gpu_group_simulate_parallel(g_, &soa.view, &c, subs.data(), subs.size(),
                                            fetch.empty() ? nullptr : fetch.data(), &tot));
    return detail::to_result(trace.size(), subs, tot, std::move(fetch));
  }

private:
  void check(int rc) {
    if (rc != 0) throw Error(ilsim_gpu_group_last_error(g_));
  }
  ilsim_gpu_group* g_ = nullptr;
};

// Multi-GPU drop-in: the partition sharded over `devices`.
inline ParallelResult simulate_parallel_gpu(std::span<const AnnotatedInstruction> trace, const ModelWeights& w,
                                            const ParallelConfig& config, const std::vector<int>& devices,
                                            int precision = ILSIM_PREC_TF32X3) {
  Group g(devices, precision);
  g.load_model(w);
  return g.simulate_parallel(trace, config);
}

// Secondary drop-in behind the reference's plugin interface
// (LatencyPredictor, predictor.hpp:19-29): CnnPredictor with K2 + decode on
// the GPU, for callers that keep the reference's host round loop
// (teacher-forced use, simcore.cpp:185-196 with a GPU predictor).
class CudaCnnPredictor final : public LatencyPredictor {
public:
  explicit CudaCnnPredictor(ModelWeights weights, int device = 0, int precision = ILSIM_PREC_TF32X3)
      : weights_(std::move(weights)), ctx_(device, precision) {
    ctx_.load_model(weights_);
  }
  int max_context() const override { return weights_.config.max_context; }
  const NormStats* norm_stats() const override { return &weights_.norm; }
  void predict(std::span<const PredictRequest> requests, std::span<LatencyTriple> out) override {
    ctx_.predict(requests, out);
  }

private:
  ModelWeights weights_;
  Context ctx_;
};

}  // namespace ilsim::gpu
