// TEST INFRASTRUCTURE ONLY — the CPU oracle ("port") for the SimNet parallel
// sub-trace simulation path.  It is the checker for the CUDA product and is
// itself pinned against the reference library (oracle/_ref) and the
// reference's golden cases (tests/test_oracle_*.py).  Only tests/, smoke()
// and bench.py's cpu_baseline leg may load it.
#pragma once
#include <cstdint>

extern "C" {

// Structure-of-arrays view of an annotated trace (trace.hpp:49-109 fields the
// simulate path reads).  truth may be null unless oracle mode is requested.
struct port_trace {
  uint64_t n;
  const uint64_t* pc;         // [n]
  const uint8_t* op;          // [n][13]
  const uint16_t* src;        // [n][8]
  const uint16_t* dst;        // [n][6]
  const uint8_t* has_data;    // [n]
  const uint64_t* data_addr;  // [n]
  const uint16_t* hist;       // [n][14]
  const uint32_t* truth;      // [n][3] fetch, execution, store
};

// CnnConfig (cnn.hpp:17-40) + NormStats (dataset.hpp:54-65) + params.
struct port_model {
  int32_t input_channels, max_context, sequence_length, n_conv;
  int32_t conv[8];
  int32_t fc_hidden, class_fetch, class_exec, class_store, residual;
  const double* norm;   // mean[50], stdev[50], label_mean[3], label_stdev[3]
  const float* params;  // param_count floats, reference (column-major) order
  uint64_t n_params;
};

// ParallelConfig (parallel.hpp:24-29) + SimConfig (simcore.hpp:13-20) + the
// two extensions that have no reference implementation (warm-up, drain-trim).
struct port_config {
  uint64_t k, subtrace_size, batch_max;
  int32_t max_context;          // <= 0: the model's
  uint32_t retire_bandwidth;
  int32_t per_cycle_advance;
  int32_t record_fetch;
  int32_t sequential;           // 1: simulate_trace semantics (one core, no partition)
  int32_t oracle;               // 1: truth latencies (OraclePredictor), no input build
  int32_t truth_with_inputs;    // 1: truth latencies but inputs built (input parity)
  uint32_t line_size, page_size;
  uint64_t warmup;              // extension: instructions replayed before each sub-trace
  int32_t drain_trim;           // extension: only the last sub-trace's drain is counted
  int32_t threads;              // OpenMP threads for the forward, <= 0: default
};

// Per sub-trace: instructions, total, sum_fetch, delta, drain, overflow, empty.
struct port_sub {
  uint64_t instructions, total_cycles, sum_fetch, delta, drain_cycles, overflow_stall_cycles, empty;
};

// Optional request capture (teacher forcing): request r in issue order.
struct port_capture {
  uint64_t cap;        // rows available
  uint64_t count;      // rows produced (may exceed cap; extra rows dropped)
  float* inputs;       // [cap][50*(max_context+1)] or null
  float* outputs;      // [cap][output_dim] or null (CNN mode only)
  uint64_t* index;     // [cap] trace index
  uint8_t* is_store;   // [cap]
  uint32_t* triples;   // [cap][3]
  uint32_t* round;     // [cap] round number
};

int port_simulate(const port_trace* t, const port_model* m, const port_config* c, port_sub* subs,
                  uint64_t sub_cap, uint32_t* predicted_fetch, uint64_t* totals, port_capture* cap,
                  char* err, int errlen);
int port_forward(const port_model* m, const float* inputs, uint64_t n, const uint8_t* is_store,
                 float* outputs, uint32_t* triples, char* err, int errlen);
// decode_hybrid on caller head outputs (cnn.cpp:406-417); m supplies class
// counts and label NormStats only.
int port_decode(const port_model* m, const float* outputs, uint64_t n, const uint8_t* is_store,
                uint32_t* triples);
int port_partition(uint64_t n, uint64_t k, uint64_t* starts, char* err, int errlen);
uint64_t port_model_flops(const port_model* m);
uint64_t port_param_count(const port_model* m);
int port_init_weights(port_model* m, uint64_t seed, float* params_out, char* err, int errlen);
}
