/*
 * ilsim_gpu.h — C-ABI of the B200-native SimNet parallel sub-trace simulator.
 *
 * Drop-in boundary for the reference's simulate path (reference root:
 * /root/reference/proj).  Every entry point below replaces one reference
 * interface; the citation names the file:line it stands in for.  Plain
 * pointers and sizes only — no C++ or torch types cross this boundary.  All
 * functions that can fail return int (0 = ok); the message is available from
 * ilsim_gpu_last_error(ctx) (or the err buffer for context-free calls) and
 * mirrors the reference's ilsim::Error text (common.hpp:12-15), e.g.
 * "batch_max must be >= 1" (parallel.cpp:40).
 *
 * Threading: one context per GPU, one caller per context (the reference calls
 * predict from one thread, parallel.cpp:70-75).  Multi-GPU, either
 *  - one process per GPU, each simulating a contiguous shard of the global
 *    partition (ilsim_sim_config.shard_*) from its own slice of the trace
 *    (ilsim_trace_view.base); the caller sums the totals (NCCL all-reduce), or
 *  - one process, several GPUs: ilsim_gpu_group_* (one host thread per
 *    device inside the library, results gathered in sub-trace order).
 */
#ifndef ILSIM_GPU_H_
#define ILSIM_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ILSIM_GPU_ABI_VERSION 2

typedef struct ilsim_gpu_ctx ilsim_gpu_ctx;

/* Inference arithmetic for the latency predictor (K2).
 * FP32   : SIMT fp32 FFMA (exact fp32 products, order differs from Eigen).
 * TF32X3 : tcgen05 kind::tf32 with the 3-term hi/lo split (fp32-faithful).
 * TF32   : tcgen05 kind::tf32, one pass.
 * BF16   : tcgen05 kind::f16 with bf16 operands, fp32 accumulate.
 * FP8    : tcgen05 kind::f8f6f4, e4m3 activations and weights (per-layer
 *          power-of-two weight scale), fp32 accumulate and fp32 FC tail.
 *          Fused simulate path only (no teacher-forced predict, no unfused
 *          rounds); its CPI error is reported, not bounded.                 */
enum {
  ILSIM_PREC_FP32 = 0,
  ILSIM_PREC_TF32X3 = 1,
  ILSIM_PREC_TF32 = 2,
  ILSIM_PREC_BF16 = 3,
  ILSIM_PREC_FP8 = 4
};

typedef struct ilsim_gpu_options {
  int32_t device;    /* CUDA device ordinal owned by this context            */
  int32_t precision; /* ILSIM_PREC_*                                          */
  int32_t reserved[6];
} ilsim_gpu_options;

/* Structure-of-arrays view of an annotated trace: the AnnotatedInstruction
 * fields the simulate path reads (trace.hpp:49-109).  truth is only needed
 * in oracle mode (OraclePredictor, predictor.hpp:45-59).
 * n is the GLOBAL trace length (the partition is computed over it); the
 * arrays hold instructions [base, base + rows) of that trace, so a process
 * simulating one shard of a large trace passes only its slice (rows must
 * cover the shard's instructions plus its warm-up prefix).  base = 0: the
 * arrays hold the whole trace.  (ABI v2 added base.)                      */
typedef struct ilsim_trace_view {
  uint64_t n;
  const uint64_t* pc;        /* [n]                                  */
  const uint8_t* op;         /* [n][13] StaticInstruction::op        */
  const uint16_t* src;       /* [n][8]                               */
  const uint16_t* dst;       /* [n][6]                               */
  const uint8_t* has_data;   /* [n]                                  */
  const uint64_t* data_addr; /* [n]                                  */
  const uint16_t* hist;      /* [n][14] HistoryFeatures::v           */
  const uint32_t* truth;     /* [n][3] fetch, execution, store       */
  uint64_t base;             /* global index of the arrays' row 0    */
} ilsim_trace_view;

/* CnnConfig (cnn.hpp:17-40).                                                 */
typedef struct ilsim_cnn_config {
  int32_t input_channels, max_context, sequence_length, n_conv;
  int32_t conv[8];
  int32_t fc_hidden, class_fetch, class_exec, class_store, residual;
} ilsim_cnn_config;

/* ParallelConfig (parallel.hpp:24-29) + SimConfig (simcore.hpp:13-20), plus
 * sharding and two extensions with no reference implementation.            */
typedef struct ilsim_sim_config {
  uint64_t k;             /* sub-traces (0 = derive from subtrace_size)             */
  uint64_t subtrace_size; /* 0 = derive from k; both set must agree (parallel.cpp:30-38) */
  uint64_t batch_max;     /* >= 1; validated, results are batch-independent          */
  int32_t max_context;    /* <= 0: the model's (cmd_simulate, ilsim_main.cpp:141)    */
  uint32_t retire_bandwidth;
  int32_t per_cycle_advance;
  int32_t record_fetch;
  int32_t sequential;     /* 1: simulate_trace (simcore.hpp:94-95)                    */
  int32_t oracle;         /* 1: truth latencies (OraclePredictor), no model needed    */
  uint32_t line_size, page_size;
  uint64_t warmup;        /* extension: preceding instructions replayed, not counted */
  int32_t drain_trim;     /* extension: only the last sub-trace's drain is counted   */
  int32_t write_ring;     /* write-queue ring entries per sub-trace (0 = 2048)       */
  uint64_t shard_begin;   /* this process simulates sub-traces [shard_begin,        */
  uint64_t shard_end;     /*   shard_end) of the global partition; 0,0 = all        */
  /* reserved[0]: 1 = per-kernel event timing (no graphs, diagnostics);
   * reserved[1]: 1 = oracle latencies but inputs still gathered (input-parity
   * test hook; the reference's OraclePredictor builds none, simcore.cpp:32);
   * reserved[2]: 1 = unfused tensor-core round (separate K1 kernel + TMA conv
   * chain) instead of the fused round front (A/B diagnostics). */
  int32_t reserved[4];
} ilsim_sim_config;

/* SimResult (simcore.hpp:22-32) without the fetch series.                    */
typedef struct ilsim_sub_result {
  uint64_t instructions, total_cycles, sum_fetch, delta, drain_cycles, overflow_stall_cycles, empty;
} ilsim_sub_result;

/* ParallelResult aggregate (parallel.hpp:31-38) for the simulated shard.     */
typedef struct ilsim_totals {
  uint64_t sub_traces, instructions, total_cycles, sum_fetch, delta, drain_cycles,
      overflow_stall_cycles, rounds;
  double cpi;
  double device_ms;       /* CUDA-event time of the round loop (inputs resident)    */
  double kernel_ms[4];    /* per-kernel event time: context, inference, decode, pack */
  uint64_t launches;      /* kernels launched by the round loop                     */
} ilsim_totals;

/* ---- context (replaces constructing CnnPredictor, predictor.cpp:9-11) ---- */
int ilsim_gpu_create(const ilsim_gpu_options* opts, ilsim_gpu_ctx** out, char* err, int errlen);
void ilsim_gpu_destroy(ilsim_gpu_ctx* ctx);
const char* ilsim_gpu_last_error(const ilsim_gpu_ctx* ctx);
int ilsim_gpu_abi_version(void);

/* Weights + NormStats (load_model, cnn.cpp:662-697, already parsed).
 * norm = mean[50], stdev[50], label_mean[3], label_stdev[3].                 */
int ilsim_gpu_load_model(ilsim_gpu_ctx* ctx, const ilsim_cnn_config* cfg, const double* norm,
                         const float* params, uint64_t n_params);

/* Upload the instructions this shard needs (trace.cpp:102-124 output).       */
int ilsim_gpu_load_trace(ilsim_gpu_ctx* ctx, const ilsim_trace_view* trace,
                         const ilsim_sim_config* cfg);

/* GPU trace ingest: the same, straight from the SNT1 record bytes (the file
 * body after its 24-byte header, trace.cpp:49-83 / 102-124).  The shard's
 * 108-byte records are copied to the device and unpacked there (read_record
 * semantics: address and size are zero without data); the host does no
 * per-record work.  with_truth: also keep the recorded latencies (oracle).   */
int ilsim_gpu_load_trace_records(ilsim_gpu_ctx* ctx, const void* records, uint64_t n,
                                 const ilsim_sim_config* cfg, int32_t with_truth);

/* Round loop over the loaded trace (simulate_parallel, parallel.cpp:26-93, or
 * simulate_trace, simcore.cpp:185-196, when cfg->sequential).
 * subs: one per simulated sub-trace (shard); predicted_fetch: per owned
 * instruction of the shard in trace order (may be NULL).                      */
int ilsim_gpu_run(ilsim_gpu_ctx* ctx, const ilsim_sim_config* cfg, ilsim_sub_result* subs,
                  uint64_t sub_cap, uint32_t* predicted_fetch, ilsim_totals* totals);

/* load_trace + run: the one-call drop-in for simulate_parallel.              */
int ilsim_gpu_simulate_parallel(ilsim_gpu_ctx* ctx, const ilsim_trace_view* trace,
                                const ilsim_sim_config* cfg, ilsim_sub_result* subs,
                                uint64_t sub_cap, uint32_t* predicted_fetch, ilsim_totals* totals);

/* Batched inference + hybrid decode on caller inputs (n x 50*(max_context+1)
 * floats, the PredictRequest::input layout): CnnPredictor::predict
 * (predictor.cpp:13-29).  outputs: n x output_dim raw head values (may be
 * NULL); triples: n x {fetch, execution, store}.                              */
int ilsim_gpu_predict(ilsim_gpu_ctx* ctx, const float* inputs, uint64_t n, const uint8_t* is_store,
                      float* outputs, uint32_t* triples);

/* ---- multi-device group (one process, several GPUs) -------------------------
 * simulate_parallel (parallel.hpp:43-44) over a list of devices: the library
 * owns one context and one host thread per device, shards the global
 * partition contiguously (device i gets sub-traces [i*k/n ...), the first
 * k % n devices one more), uploads each device only its slice of the view,
 * and returns every sub-result in sub-trace order plus the summed totals
 * (device_ms = the slowest device).  Results are identical for any device
 * list (test_parallel.cpp:114-146).  A device may appear more than once (its
 * shards then run concurrently on separate streams).                         */
typedef struct ilsim_gpu_group ilsim_gpu_group;
int ilsim_gpu_group_create(const ilsim_gpu_options* opts, const int32_t* devices, int32_t n_devices,
                           ilsim_gpu_group** out, char* err, int errlen);
void ilsim_gpu_group_destroy(ilsim_gpu_group* group);
const char* ilsim_gpu_group_last_error(const ilsim_gpu_group* group);
int ilsim_gpu_group_size(const ilsim_gpu_group* group);
int ilsim_gpu_group_load_model(ilsim_gpu_group* group, const ilsim_cnn_config* cfg, const double* norm,
                               const float* params, uint64_t n_params);
int ilsim_gpu_group_simulate_parallel(ilsim_gpu_group* group, const ilsim_trace_view* trace,
                                      const ilsim_sim_config* cfg, ilsim_sub_result* subs, uint64_t sub_cap,
                                      uint32_t* predicted_fetch, ilsim_totals* totals);

/* Test hook: hybrid decode (decode_hybrid, cnn.cpp:388-417) of caller head
 * outputs (n x output_dim floats, the ilsim_gpu_predict output layout) with
 * the loaded model's NormStats label statistics and head sizes.  path 0: the
 * per-thread decode of the unfused / teacher-forced path (decode.cuh);
 * path 1: the warp-cooperative decode of the fused round (fc_decode.cuh).
 * Lets the reference's decode goldens (test_cnn.cpp:183-224) run on the
 * device functions themselves.                                              */
int ilsim_gpu_decode_outputs(ilsim_gpu_ctx* ctx, const float* outputs, uint64_t n, const uint8_t* is_store,
                             uint32_t* triples, int32_t path);

/* Test hook: capture the gathered input tensor of round `round` of the next
 * run (k x 50*(max_context+1) floats in sub-trace order; rows of inactive
 * sub-traces untouched).  round = UINT32_MAX disables.                        */
int ilsim_gpu_set_capture(ilsim_gpu_ctx* ctx, uint32_t round, float* inputs, uint64_t rows);

/* ---- context-free helpers --------------------------------------------------*/
/* partition (parallel.cpp:9-24): starts[k].                                   */
int ilsim_gpu_partition(uint64_t n, uint64_t k, uint64_t* starts, char* err, int errlen);
/* model_flops (cnn.cpp:319-333): multiplications per forward.                 */
uint64_t ilsim_gpu_model_flops(const ilsim_cnn_config* cfg);
/* param_count (cnn.cpp:317).                                                  */
uint64_t ilsim_gpu_param_count(const ilsim_cnn_config* cfg);
/* init_weights (cnn.cpp:335-352) parameter draw.                              */
int ilsim_gpu_init_weights(const ilsim_cnn_config* cfg, uint64_t seed, float* params, uint64_t n,
                           char* err, int errlen);

#ifdef __cplusplus
}
#endif
#endif /* ILSIM_GPU_H_ */
