// Shared device-side definitions for the SimNet sub-trace simulator (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace simnet {

constexpr int kSlots = 50;        // FeatureLayout::kSlots (trace.hpp:113)
constexpr int kStatic = 41;       // op 13 + src 8 + dst 6 + history 14 (trace.hpp:115-118)
constexpr int kStatStride = 48;   // floats per instruction in the packed static table
constexpr int kSlotResidence = 41, kSlotExecution = 42, kSlotStore = 43, kSlotFlag0 = 44,
              kSlotReserved = 49;

// Instruction flag bits in the packed trace.
constexpr uint8_t kFlagMem = 1, kFlagStore = 2;

// Sub-trace status codes (device -> host error reporting).
enum : uint32_t { kOk = 0, kErrStall = 1, kErrDrain = 2, kErrWriteRing = 3 };

// One in-flight instruction (SimCore::InFlight, simcore.hpp:61-68) in the
// push-tick formulation: residence == cur - push (simcore.hpp:55-57), so no
// per-entry counter is stored and "advance" is O(1).  Normalised
// execution/store slots are computed once at push, and the instruction's pc /
// data address / flags ride along so the gather needs no extra load level
// for the dependency flags.  48 B.
struct __align__(16) RingEntry {
  uint64_t push;      // cur_tick when pushed
  uint64_t pc;        // StaticInstruction::pc
  uint64_t addr;      // StaticInstruction::data_addr
  uint32_t idx;       // position within the sub-trace (local_index)
  uint32_t exec;      // predicted execution latency
  uint32_t store;     // predicted store latency
  float nexec;        // normalised slot 42
  float nstore;       // normalised slot 43
  uint32_t flags;     // kFlagMem | kFlagStore
};
static_assert(sizeof(RingEntry) == 48, "RingEntry layout");

// Per-sub-trace machine state (SimCore members, simcore.hpp:79-90, plus the
// round-loop bookkeeping of parallel.cpp:63-81).  128 B.
struct __align__(16) SubState {
  uint64_t cur, sum_fetch, overflow, drain;
  uint64_t base_cur, base_overflow;  // warm-up extension: counters at warm-up end
  uint64_t begin;                    // device-local index of the first simulated instruction
  uint64_t fetch_off;                // offset of the first owned instruction in predicted_fetch
  uint32_t len, warm, pos;           // simulated length, warm-up prefix, next instruction
  uint32_t pend_f, pend_e, pend_s, has_pend;
  uint32_t ph, pt, wh, wt;           // proc / write ring head, tail (monotonic counters)
  uint32_t status;
  uint32_t count_drain;
  uint32_t xcols;                    // gathered-input columns written last round (zeroing bound)
  uint64_t err_tick;
  uint64_t t_pc, t_addr;             // pc / data address of instruction `pos` (set by the gather)
  uint32_t t_flags;                  // its flags, copied into the ring entry at push
  uint32_t awaiting;                 // fused round: input gathered, prediction not yet decoded
  uint32_t pad_[2];
};
static_assert(sizeof(SubState) == 160, "SubState layout");

// Normalisation constants derived from NormStats (dataset.hpp:54-65).
struct NormConsts {
  double mean[kSlots];
  double sd[kSlots];
  double label_mean[3];
  double label_sd[3];
  float zero[kSlots];   // normalised raw 0 per slot
  float one[kSlots];    // normalised raw 1 per slot (dependency flags)
};

// f32(clamp((raw - mean)/sd, -10, 10)) exactly as simcore.cpp:43-44: fp64
// subtract and IEEE divide (no contraction), clamp, round to f32.
__host__ __device__ inline float norm_slot(int32_t raw, double mean, double sd) {
#ifdef __CUDA_ARCH__
  const double z = __ddiv_rn(__dsub_rn(static_cast<double>(raw), mean), sd);
#else
  volatile double d = static_cast<double>(raw) - mean;
  const double z = d / sd;
#endif
  const double c = z < -10.0 ? -10.0 : (z > 10.0 ? 10.0 : z);
  return static_cast<float>(c);
}

}  // namespace simnet
