// TEST INFRASTRUCTURE: the C++ drop-in (include/ilsim_gpu.hpp) driven from
// the reference's own types and round loop, as a reference maintainer would
// call it.  Linked against oracle/_ref/libilsim_ref.so (the reference's
// sources compiled unmodified + the restated forward) and libilsim_gpu.so;
// built by `make -C oracle dropin`, run by tests/test_lib.py on the GPU box.
//
//   ilsim_dropin <trace> <model> <k> <precision 0-4> [devices...]
//
// Runs on the same trace / weights / config and prints one JSON object:
//   cpu     reference simulate_parallel with its CnnPredictor (parallel.cpp:26-93)
//   plugin  reference simulate_parallel with CudaCnnPredictor plugged in
//           (LatencyPredictor, predictor.hpp:19-29: K2 + decode on the GPU)
//   gpu     ilsim::gpu::simulate_parallel_gpu (the whole loop on the GPU)
//   group   simulate_parallel_gpu over the device list (ilsim_gpu_group_*)
//   oracle  OraclePredictor on the CPU vs Context::simulate_parallel(oracle) (exact)
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "ilsim/cnn.hpp"
#include "ilsim/parallel.hpp"
#include "ilsim/predictor.hpp"
#include "ilsim/trace.hpp"
#include "ilsim_gpu.hpp"

using namespace ilsim;

static void put(const char* name, const ParallelResult& r, const ParallelResult& ref, bool last = false) {
  size_t same_subs = 0, same_fetch = 0;
  for (size_t i = 0; i < r.sub_results.size() && i < ref.sub_results.size(); ++i)
    same_subs += r.sub_results[i].total_cycles == ref.sub_results[i].total_cycles &&
                 r.sub_results[i].drain_cycles == ref.sub_results[i].drain_cycles &&
                 r.sub_results[i].overflow_stall_cycles == ref.sub_results[i].overflow_stall_cycles;
  for (size_t i = 0; i < r.predicted_fetch.size() && i < ref.predicted_fetch.size(); ++i)
    same_fetch += r.predicted_fetch[i] == ref.predicted_fetch[i];
  std::printf("\"%s\": {\"total_cycles\": %llu, \"instructions\": %llu, \"subs\": %zu, \"same_subs\": %zu, "
              "\"fetch\": %zu, \"same_fetch\": %zu}%s\n",
              name, static_cast<unsigned long long>(r.total_cycles), static_cast<unsigned long long>(r.instructions),
              r.sub_results.size(), same_subs, r.predicted_fetch.size(), same_fetch, last ? "" : ",");
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s trace model k precision [devices...]\n", argv[0]);
    return 2;
  }
  try {
    const Trace trace = read_trace(argv[1]);
    const ModelWeights w = load_model(argv[2]);
    const int precision = std::atoi(argv[4]);
    std::vector<int> devices;
    for (int i = 5; i < argc; ++i) devices.push_back(std::atoi(argv[i]));
    if (devices.empty()) devices = {0};
    ParallelConfig pc;
    pc.k = std::strtoull(argv[3], nullptr, 10);
    pc.sim.max_context = w.config.max_context;

    CnnPredictor cpu_pred(w);
    const ParallelResult cpu = simulate_parallel(trace.instructions, cpu_pred, pc);
    gpu::CudaCnnPredictor gpu_pred(w, devices[0], precision);
    const ParallelResult plugin = simulate_parallel(trace.instructions, gpu_pred, pc);
    const ParallelResult whole = gpu::simulate_parallel_gpu(trace.instructions, w, pc, devices[0], precision);
    const ParallelResult group = gpu::simulate_parallel_gpu(trace.instructions, w, pc, devices, precision);
    OraclePredictor oracle_pred(trace.instructions);
    ParallelConfig po = pc;
    const ParallelResult oracle_cpu = simulate_parallel(trace.instructions, oracle_pred, po);
    gpu::Context ctx(devices[0], precision);
    const ParallelResult oracle_gpu = ctx.simulate_parallel(trace.instructions, po, /*oracle=*/true);
    std::printf("{\n");
    put("cpu", cpu, cpu);
    put("plugin", plugin, cpu);
    put("gpu", whole, cpu);
    put("group", group, whole);
    put("oracle_cpu", oracle_cpu, oracle_cpu);
    put("oracle_gpu", oracle_gpu, oracle_cpu, true);
    std::printf("}\n");
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 1;
  }
  return 0;
}
