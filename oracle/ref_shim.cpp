// TEST INFRASTRUCTURE ONLY — C-ABI shim over the reference library built from
// /root/reference/proj/src (oracle/Makefile).  Used by tests/ to pin the
// oracle port against the reference's own code, by tests/golden/make_golden.py
// to produce fixtures, and by bench.py's cpu_baseline / --impl reference legs.
// Never linked into, or called by, the product path.
//
// Every entry returns 0 on success, 1 on ilsim::Error / std::exception with
// the message copied into `err` (the reference CLI prints "error: <msg>",
// tools/ilsim_main.cpp:285-288).
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "ilsim/cnn.hpp"
#include "ilsim/dataset.hpp"
#include "ilsim/des.hpp"
#include "ilsim/parallel.hpp"
#include "ilsim/predictor.hpp"
#include "ilsim/simcore.hpp"
#include "ilsim/trace.hpp"
#include "ilsim/workload.hpp"

using namespace ilsim;

namespace {

void put_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = 0;
  }
}

template <typename F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// Reference predictor wrapper that records every request it is asked for
// (input tensor, trace index, store flag) and the decoded triple it returned.
class Recorder final : public LatencyPredictor {
public:
  Recorder(LatencyPredictor& inner, const NormStats* norm_for_inputs, int max_ctx)
      : inner_(inner), norm_(norm_for_inputs), max_ctx_(max_ctx) {}
  bool needs_input() const override { return norm_ != nullptr; }
  int max_context() const override { return max_ctx_; }
  const NormStats* norm_stats() const override { return norm_; }
  void predict(std::span<const PredictRequest> req, std::span<LatencyTriple> out) override {
    inner_.predict(req, out);
    const size_t width = static_cast<size_t>(FeatureLayout::kSlots) * (max_ctx_ + 1);
    for (size_t i = 0; i < req.size(); ++i) {
      index.push_back(req[i].trace_index);
      is_store.push_back(req[i].target_is_store ? 1 : 0);
      triples.push_back(out[i]);
      if (req[i].input) inputs.insert(inputs.end(), req[i].input, req[i].input + width);
    }
  }
  std::vector<uint64_t> index;
  std::vector<uint8_t> is_store;
  std::vector<LatencyTriple> triples;
  std::vector<float> inputs;

private:
  LatencyPredictor& inner_;
  const NormStats* norm_;
  int max_ctx_;
};

// Truth latencies with inputs still built (OraclePredictor skips the input
// build, simcore.cpp:32); used for input-tensor parity.
class TruthWithInputs final : public LatencyPredictor {
public:
  TruthWithInputs(std::span<const AnnotatedInstruction> t, NormStats n, int mc)
      : t_(t), n_(n), mc_(mc) {}
  int max_context() const override { return mc_; }
  const NormStats* norm_stats() const override { return &n_; }
  void predict(std::span<const PredictRequest> req, std::span<LatencyTriple> out) override {
    for (size_t i = 0; i < req.size(); ++i) out[i] = t_[req[i].trace_index].truth;
  }

private:
  std::span<const AnnotatedInstruction> t_;
  NormStats n_;
  int mc_;
};

struct SimArgs {
  uint64_t k, subtrace_size, batch_max;
  int32_t max_context;  // <=0: model's (cmd_simulate, ilsim_main.cpp:141)
  uint32_t retire_bandwidth;
  int32_t per_cycle;
  int32_t sequential;   // 1: simulate_trace instead of simulate_parallel
  int32_t workers;      // OpenMP threads, <=0: default
};

// sub_out: per sub-trace 7 u64 {instructions,total,sum_fetch,delta,drain,overflow,empty}
void fill_sub(const SimResult& r, uint64_t* o) {
  o[0] = r.instructions;
  o[1] = r.total_cycles;
  o[2] = r.sum_fetch;
  o[3] = r.delta;
  o[4] = r.drain_cycles;
  o[5] = r.overflow_stall_cycles;
  o[6] = r.empty ? 1 : 0;
}

}  // namespace

extern "C" {

int ref_make_trace(const char* kind, uint64_t n, uint64_t seed, uint64_t footprint,
                   const char* out_path, uint64_t* des_total, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    WorkloadSpec spec;
    spec.kind = workload_kind_from_string(kind);
    spec.op_class_mix = WorkloadSpec::default_mix(spec.kind);
    spec.instruction_count = n;
    spec.seed = seed;
    spec.memory_footprint_bytes = footprint;
    const DesResult res = des_simulate(generate(spec), ProcessorConfig{});
    write_trace(out_path, res.trace);
    if (des_total) *des_total = res.total_cycles;
  });
}

// Model with the reference's init rule.  NormStats either identity
// (identity_norm=1, as test_parallel.cpp:121) or compute_norm_stats over a
// dataset built from `trace_path` (dataset.cpp:243-274).
int ref_make_model(const char* trace_path, int32_t max_context, const int32_t* conv, int32_t nconv,
                   int32_t fc_hidden, int32_t residual, uint64_t seed, int32_t identity_norm,
                   const char* out_path, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    CnnConfig cfg = CnnConfig::preset_c3(max_context);
    cfg.conv_channels.assign(conv, conv + nconv);
    cfg.fc_hidden = fc_hidden;
    cfg.residual_blocks = residual != 0;
    NormStats norm;
    if (!identity_norm) {
      const Trace t = read_trace(trace_path);
      FeatureLayout layout{max_context};
      const Dataset ds = build_dataset({&t.instructions}, layout, true, SplitRatios{});
      norm = ds.norm;
    }
    save_model(out_path, init_weights(cfg, norm, seed));
  });
}

int ref_simulate(const char* trace_path, const char* model_path, const SimArgs* a,
                 uint64_t* sub_out, uint64_t sub_cap, uint32_t* predicted_fetch,
                 uint64_t* totals, double* seconds, char* err, int errlen) {
  return guarded(err, errlen, [&] {
#ifdef _OPENMP
    if (a->workers > 0) omp_set_num_threads(a->workers);
#endif
    const Trace trace = read_trace(trace_path);
    std::unique_ptr<LatencyPredictor> pred;
    SimConfig sim;
    sim.retire_bandwidth = a->retire_bandwidth;
    sim.per_cycle_advance = a->per_cycle != 0;
    if (!model_path || !*model_path) {
      pred = std::make_unique<OraclePredictor>(trace.instructions);
      if (a->max_context > 0) sim.max_context = a->max_context;
    } else {
      auto cnn = std::make_unique<CnnPredictor>(load_model(model_path));
      sim.max_context = a->max_context > 0 ? a->max_context : cnn->max_context();
      pred = std::move(cnn);
    }
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<SimResult> subs;
    uint64_t total = 0;
    if (a->sequential) {
      subs.push_back(simulate_trace(trace.instructions, *pred, sim));
      total = subs[0].total_cycles;
    } else {
      ParallelConfig pc;
      pc.k = a->k;
      pc.subtrace_size = a->subtrace_size;
      pc.batch_max = a->batch_max;
      pc.sim = sim;
      ParallelResult pr = simulate_parallel(trace.instructions, *pred, pc);
      subs = std::move(pr.sub_results);
      total = pr.total_cycles;
    }
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (subs.size() > sub_cap) throw Error("shim: sub_cap too small");
    size_t off = 0;
    for (size_t i = 0; i < subs.size(); ++i) {
      fill_sub(subs[i], sub_out + 7 * i);
      if (predicted_fetch) {
        std::copy(subs[i].predicted_fetch.begin(), subs[i].predicted_fetch.end(), predicted_fetch + off);
        off += subs[i].predicted_fetch.size();
      }
    }
    totals[0] = subs.size();
    totals[1] = total;
    totals[2] = trace.instructions.size();
  });
}

// Records the request stream of simulate_parallel (or simulate_trace when
// a->sequential).  mode 0: CNN model; mode 1: truth latencies with inputs
// built using the model file's NormStats.  Outputs hold `cap` requests.
int ref_capture(const char* trace_path, const char* model_path, int32_t mode, const SimArgs* a,
                uint64_t cap, float* inputs, uint64_t* index, uint8_t* is_store,
                uint32_t* triples, uint64_t* count, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const Trace trace = read_trace(trace_path);
    const ModelWeights w = load_model(model_path);
    SimConfig sim;
    sim.retire_bandwidth = a->retire_bandwidth;
    sim.per_cycle_advance = a->per_cycle != 0;
    sim.max_context = a->max_context > 0 ? a->max_context : w.config.max_context;
    CnnPredictor cnn(w);
    TruthWithInputs truth(trace.instructions, w.norm, sim.max_context);
    LatencyPredictor& inner = mode == 0 ? static_cast<LatencyPredictor&>(cnn) : truth;
    Recorder rec(inner, &w.norm, sim.max_context);
    if (a->sequential) {
      simulate_trace(trace.instructions, rec, sim);
    } else {
      ParallelConfig pc;
      pc.k = a->k;
      pc.subtrace_size = a->subtrace_size;
      pc.batch_max = a->batch_max;
      pc.sim = sim;
      simulate_parallel(trace.instructions, rec, pc);
    }
    const size_t width = static_cast<size_t>(FeatureLayout::kSlots) * (sim.max_context + 1);
    const uint64_t n = std::min<uint64_t>(cap, rec.index.size());
    for (uint64_t i = 0; i < n; ++i) {
      if (inputs) std::memcpy(inputs + i * width, rec.inputs.data() + i * width, width * 4);
      index[i] = rec.index[i];
      is_store[i] = rec.is_store[i];
      triples[3 * i + 0] = rec.triples[i].fetch;
      triples[3 * i + 1] = rec.triples[i].execution;
      triples[3 * i + 2] = rec.triples[i].store;
    }
    *count = rec.index.size();
  });
}

// Reference forward + decode on caller-provided inputs (n x model width).
int ref_forward(const char* model_path, const float* inputs, uint64_t n, const uint8_t* is_store,
                float* outputs, uint32_t* triples, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const ModelWeights w = load_model(model_path);
    const size_t width = static_cast<size_t>(FeatureLayout::kSlots) * (w.config.max_context + 1);
    const int od = w.config.output_dim();
    CnnWorkspace ws;
    for (uint64_t i = 0; i < n; ++i) {
      const PredictionOutput po = forward(w, inputs + i * width, ws);
      float* y = outputs + i * od;
      for (int j = 0; j < 3; ++j) y[j] = po.regression[j];
      std::copy(po.fetch_logits.begin(), po.fetch_logits.end(), y + 3);
      std::copy(po.exec_logits.begin(), po.exec_logits.end(), y + 3 + po.fetch_logits.size());
      std::copy(po.store_logits.begin(), po.store_logits.end(),
                y + 3 + po.fetch_logits.size() + po.exec_logits.size());
      const LatencyTriple t = decode_hybrid(po, w.norm, is_store[i] != 0);
      triples[3 * i + 0] = t.fetch;
      triples[3 * i + 1] = t.execution;
      triples[3 * i + 2] = t.store;
    }
  });
}

int ref_partition(uint64_t n, uint64_t k, uint64_t* starts, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const PartitionPlan p = partition(n, k);
    std::copy(p.starts.begin(), p.starts.end(), starts);
  });
}

uint64_t ref_model_flops_c3(int32_t residual) {
  CnnConfig c = CnnConfig::preset_c3();
  c.residual_blocks = residual != 0;
  return model_flops(c);
}

}  // extern "C"
