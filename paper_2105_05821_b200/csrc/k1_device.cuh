// K1 device building blocks shared by the standalone context kernel
// (sim_kernels.cu) and the fused round-front kernel (round_front.cu):
// SimCore::retire / apply_step / drain on the push-tick ring state
// (simcore.cpp:68-159) and the per-column context descriptor of
// next_request (simcore.cpp:25-66, dataset.cpp:47-75).
#pragma once
#include "common.cuh"

namespace simnet {

namespace k1 {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t leading_run(uint32_t mask) {
  return mask == kFull ? 32u : static_cast<uint32_t>(__ffs(~mask) - 1);
}

struct Rings {
  RingEntry* proc;
  RingEntry* wq;
  uint32_t pmask, wmask, wcap;
};

__device__ __forceinline__ Rings rings_of(RingEntry* proc, RingEntry* wq, uint32_t pmask, uint32_t wmask,
                                          uint64_t s) {
  return Rings{proc + s * (pmask + 1ull), wq + s * (wmask + 1ull), pmask, wmask, wmask + 1u};
}

// SimCore::retire (simcore.cpp:68-84).  Warp-uniform in/out; returns the
// number of queue transitions.  Sets *err on write-ring overflow.  In-order
// retirement of the proc queue is the run of leading ready entries (ballot);
// stores move to the write queue by ballot/popc compaction.
__device__ inline uint32_t warp_retire(uint64_t cur, uint64_t budget, const Rings& r, uint32_t& ph, uint32_t pt,
                                       uint32_t& wh, uint32_t& wt, uint32_t* err) {
  const uint32_t lane = lane_id();
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t events = 0;
  while (budget > 0 && ph != pt) {
    const uint32_t n = min(pt - ph, 32u);
    RingEntry e;
    bool ready = false;
    if (lane < n) {
      e = r.proc[(ph + lane) & r.pmask];
      ready = (cur - e.push) >= e.exec;
    }
    const uint32_t run = leading_run(__ballot_sync(kFull, ready));
    const uint32_t take = static_cast<uint32_t>(min(static_cast<uint64_t>(run), budget));
    const bool mv = lane < take && (e.flags & kFlagStore);
    const uint32_t sm = __ballot_sync(kFull, mv);
    const uint32_t nmv = __popc(sm);
    if (wt + nmv - wh > r.wcap) {
      *err = kErrWriteRing;
      return events;
    }
    if (mv) r.wq[(wt + __popc(sm & lt)) & r.wmask] = e;
    wt += nmv;
    ph += take;
    budget -= take;
    events += take;
    if (take < n) break;
  }
  while (wh != wt) {
    const uint32_t n = min(wt - wh, 32u);
    bool ready = false;
    if (lane < n) {
      const RingEntry& e = r.wq[(wh + lane) & r.wmask];
      ready = (cur - e.push) >= e.store;
    }
    const uint32_t run = leading_run(__ballot_sync(kFull, ready));
    wh += run;
    events += run;
    if (run < n) break;
  }
  __syncwarp();
  return events;
}

// readiness gap of a head entry (simcore.cpp:95-110 per queue)
__device__ __forceinline__ uint64_t head_gap(uint64_t cur, uint64_t push, uint32_t lat) {
  const uint64_t res = cur - push;
  return lat > res ? lat - res : 1;
}

struct ApplyArgs {
  uint32_t bw;            // SimConfig::retire_bandwidth
  int32_t max_context;    // proc queue capacity
  int32_t per_cycle;      // SimConfig::per_cycle_advance (test mode)
  int32_t gather;         // 1: the target's flags were stashed by the previous gather
  const uint8_t* iflags;  // packed instruction flags (used when gather == 0)
  const NormConsts* nc;
};

// Apply the pending step decided by K3 for instruction st.pos
// (simcore.cpp:112-150 after the fetch advance, which K3 already did), then
// drain if it was the sub-trace's last step (parallel.cpp:79,
// simcore.cpp:152-159).  Whole warp, warp-uniform state; lane 0 writes the
// pushed ring entry.  Returns the (possibly error) status.
__device__ inline void apply_step(SubState& st, const Rings& r, const ApplyArgs& a) {
  const uint32_t lane = lane_id();
  uint32_t err = kOk;
  const uint32_t F = st.pend_f;
  // fetch advance: K3 already moved cur by F (lumped); retire with budget bw*F
  if (F > 0) {
    if (a.per_cycle) {
      for (uint32_t c = 0; c < F && err == kOk; ++c) {
        st.cur += 1;
        warp_retire(st.cur, a.bw, r, st.ph, st.pt, st.wh, st.wt, &err);
      }
    } else {
      warp_retire(st.cur, static_cast<uint64_t>(a.bw) * F, r, st.ph, st.pt, st.wh, st.wt, &err);
    }
  }
  // forced stall (simcore.cpp:127-136): budget bw, not bw*gap
  while (err == kOk && st.pt - st.ph >= static_cast<uint32_t>(a.max_context)) {
    const uint32_t before = st.pt - st.ph;
    const RingEntry& h = r.proc[st.ph & r.pmask];
    const uint64_t gap = head_gap(st.cur, h.push, h.exec);
    st.cur += gap;
    st.overflow += gap;
    warp_retire(st.cur, a.bw, r, st.ph, st.pt, st.wh, st.wt, &err);
    if (err == kOk && st.pt - st.ph >= before) {
      err = kErrStall;
      st.err_tick = st.cur;
    }
  }
  if (err == kOk) {  // push (simcore.cpp:138-145)
    if (lane == 0) {
      const NormConsts& nc = *a.nc;
      RingEntry e;
      e.push = st.cur;
      e.idx = st.pos;
      e.exec = st.pend_e;
      e.store = st.pend_s;
      e.nexec = norm_slot(static_cast<int32_t>(st.pend_e), nc.mean[kSlotExecution], nc.sd[kSlotExecution]);
      e.nstore = norm_slot(static_cast<int32_t>(st.pend_s), nc.mean[kSlotStore], nc.sd[kSlotStore]);
      e.pc = st.t_pc;  // stashed by this sub-trace's previous gather (0 when none ran)
      e.addr = st.t_addr;
      e.flags = a.gather ? st.t_flags : a.iflags[st.begin + st.pos];
      r.proc[st.pt & r.pmask] = e;
    }
    st.pt += 1;
    st.pos += 1;
    st.has_pend = 0;
    if (st.pos == st.warm) {  // warm-up extension: counting starts after this step
      st.base_cur = st.cur;
      st.base_overflow = st.overflow;
    }
    // drain right after the last step (parallel.cpp:79, simcore.cpp:152-159)
    if (st.pos == st.len && st.count_drain) {
      __syncwarp();  // lane 0's push above is visible to the lanes reading the queue heads below
      while (err == kOk && (st.ph != st.pt || st.wh != st.wt)) {
        uint64_t gap = ~uint64_t{0};
        if (st.ph != st.pt) {
          const RingEntry& h = r.proc[st.ph & r.pmask];
          const uint64_t g = head_gap(st.cur, h.push, h.exec);
          gap = g < gap ? g : gap;
        }
        if (st.wh != st.wt) {
          const RingEntry& h = r.wq[st.wh & r.wmask];
          const uint64_t g = head_gap(st.cur, h.push, h.store);
          gap = g < gap ? g : gap;
        }
        if (gap < 1) gap = 1;
        st.cur += gap;
        st.drain += gap;
        const uint32_t ev = warp_retire(st.cur, a.bw, r, st.ph, st.pt, st.wh, st.wt, &err);
        if (err == kOk && ev == 0) {
          err = kErrDrain;
          st.err_tick = st.cur;
        }
      }
    }
  }
  if (err != kOk) st.status = err;
  __syncwarp();
}

// memory_dependency_flags (dataset.cpp:47-60) of context entry e against the
// target (tpc, taddr, tmem): bit b = flag b.
// a / d == b / d (dataset.cpp:51-58 divides by line / page size); a power-of-two
// d (the usual 64 / 4096) is a shift instead of a 64-bit division subroutine.
__device__ __forceinline__ bool same_block(uint64_t a, uint64_t b, uint32_t d) {
  if (d != 0u && (d & (d - 1u)) == 0u) {
    const int sh = __ffs(static_cast<int>(d)) - 1;
    return (a >> sh) == (b >> sh);
  }
  return a / d == b / d;
}

__device__ __forceinline__ uint32_t dep_flags(uint64_t tpc, uint64_t taddr, bool tmem, const RingEntry& e,
                                              uint32_t line, uint32_t page) {
  uint32_t f = same_block(tpc, e.pc, line) ? 1u : 0u;
  if (tmem && (e.flags & kFlagMem)) {
    f |= (taddr == e.addr) ? 2u : 0u;
    f |= same_block(taddr, e.addr, line) ? 4u : 0u;
    f |= same_block(taddr, e.addr, page) ? 8u : 0u;
  }
  f |= same_block(tpc, e.pc, page) ? 16u : 0u;
  return f;
}

// Context column j (0-based, newest first: proc queue, then write queue).
__device__ __forceinline__ RingEntry context_entry(const SubState& st, const Rings& r, uint32_t j) {
  const uint32_t nproc = st.pt - st.ph;
  return j < nproc ? r.proc[(st.pt - 1 - j) & r.pmask] : r.wq[(st.wt - 1 - (j - nproc)) & r.wmask];
}

}  // namespace k1

}  // namespace simnet
