// TEST INFRASTRUCTURE ONLY — CPU oracle for the SimNet parallel simulation
// path; see simnet_port.hpp.  A from-scratch restatement of the reference's
// algorithm (file:line cites are relative to /root/reference/proj), written
// in the reference's own formulation (explicit per-entry residence counters,
// deques) so that it checks the CUDA product's push-tick/ring formulation
// rather than mirroring it.
#include "simnet_port.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

struct PortError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

constexpr int kSlots = 50;        // FeatureLayout::kSlots (trace.hpp:113)
constexpr int kStaticSlots = 41;  // 13 op + 8 src + 6 dst + 14 history
constexpr int kOpIsLoad = 1, kOpIsStore = 2;

// ---------------------------------------------------------------------------
// CNN (restates cnn.cpp:44-125, 219-225, 354-368, 388-417)
// ---------------------------------------------------------------------------
struct Net {
  const port_model* m;
  std::vector<size_t> w, b, p, act;
  size_t fc1_w = 0, fc1_b = 0, fc2_w = 0, fc2_b = 0, n_params = 0, act_h = 0, act_y = 0, act_n = 0;
  int out_dim = 0, flat = 0;

  explicit Net(const port_model* mm) : m(mm) {
    // n_conv == 0: the FC-only predictor (paper FC2), an extension
    // with no reference implementation: FC1 reads the unpadded input.
    if (m->n_conv < 0 || m->n_conv > 8) throw PortError("conv layer count out of range");
    out_dim = 3 + m->class_fetch + m->class_exec + m->class_store;
    flat = m->n_conv == 0 ? m->input_channels * (m->max_context + 1)
                          : m->conv[m->n_conv - 1] * (m->sequence_length >> m->n_conv);
    size_t off = 0;
    int cin = m->input_channels;
    for (int l = 0; l < m->n_conv; ++l) {
      const size_t taps = static_cast<size_t>(m->conv[l]) * 2 * cin;
      w.push_back(off);
      off += taps;
      b.push_back(off);
      off += m->conv[l];
      if (m->residual) {
        p.push_back(off);
        off += taps;
      }
      cin = m->conv[l];
    }
    fc1_w = off;
    off += static_cast<size_t>(m->fc_hidden) * flat;
    fc1_b = off;
    off += m->fc_hidden;
    fc2_w = off;
    off += static_cast<size_t>(out_dim) * m->fc_hidden;
    fc2_b = off;
    off += out_dim;
    n_params = off;
    size_t a = 0;
    int len = m->sequence_length;
    act.push_back(a);
    a += static_cast<size_t>(m->input_channels) * len;
    for (int l = 0; l < m->n_conv; ++l) {
      len >>= 1;
      act.push_back(a);
      a += static_cast<size_t>(m->conv[l]) * len;
    }
    act_h = a;
    a += m->fc_hidden;
    act_y = a;
    a += out_dim;
    act_n = a;
  }

  size_t width() const { return static_cast<size_t>(m->input_channels) * (m->max_context + 1); }

  // column-major y[rows x cols] (+)= W[rows x inner] x[inner x cols], k ascending, fused.
  static void gemm(const float* W, const float* x, float* y, int rows, int inner, int cols, bool acc) {
    for (int j = 0; j < cols; ++j) {
      float* yj = y + static_cast<size_t>(j) * rows;
      if (!acc) std::fill(yj, yj + rows, 0.0f);
      const float* xj = x + static_cast<size_t>(j) * inner;
      for (int k = 0; k < inner; ++k) {
        const float a = xj[k];
        const float* wk = W + static_cast<size_t>(k) * rows;
        for (int o = 0; o < rows; ++o) yj[o] = std::fma(wk[o], a, yj[o]);
      }
    }
  }

  // The FC-only predictor's accumulation order (no reference implementation;
  // defined here and on the GPU alike, paper_2105_05821_b200/csrc/gemm.cuh):
  // per output, an fma chain over each 512-wide K chunk starting from 0, the
  // chunk sums added in chunk order from 0.
  static void gemm_chunked(const float* W, const float* x, float* y, int rows, int inner) {
    constexpr int kChunk = 512;
    std::vector<float> acc(rows);
    std::fill(y, y + rows, 0.0f);
    for (int k0 = 0; k0 < inner; k0 += kChunk) {  // per output: the same chains, weights streamed row by row
      std::fill(acc.begin(), acc.end(), 0.0f);
      const int k1 = std::min(inner, k0 + kChunk);
      for (int k = k0; k < k1; ++k) {
        const float a = x[k];
        const float* wk = W + static_cast<size_t>(k) * rows;
        for (int o = 0; o < rows; ++o) acc[o] = std::fma(wk[o], a, acc[o]);
      }
      for (int o = 0; o < rows; ++o) y[o] += acc[o];
    }
  }

  // input: width() floats; out: out_dim floats.
  void forward(const float* input, float* out, std::vector<float>& act_buf) const {
    act_buf.resize(act_n);
    float* A = act_buf.data();
    const size_t real = width();
    const size_t padded = static_cast<size_t>(m->input_channels) * m->sequence_length;
    std::copy(input, input + real, A);
    std::fill(A + real, A + padded, 0.0f);
    const float* P = m->params;
    int cin = m->input_channels, len = m->sequence_length;
    for (int l = 0; l < m->n_conv; ++l) {
      const int cout = m->conv[l], olen = len / 2;
      const float* in = A + act[l];
      float* o = A + act[l + 1];
      gemm(P + w[l], in, o, cout, 2 * cin, olen, false);
      if (m->residual) gemm(P + p[l], in, o, cout, 2 * cin, olen, true);
      for (int j = 0; j < olen; ++j)
        for (int c = 0; c < cout; ++c) {
          float& v = o[static_cast<size_t>(j) * cout + c];
          v = std::max(v + P[b[l] + c], 0.0f);
        }
      cin = cout;
      len = olen;
    }
    float* h = A + act_h;
    if (m->n_conv == 0)
      gemm_chunked(P + fc1_w, A + act[m->n_conv], h, m->fc_hidden, flat);
    else
      gemm(P + fc1_w, A + act[m->n_conv], h, m->fc_hidden, flat, 1, false);
    for (int o = 0; o < m->fc_hidden; ++o) h[o] = std::max(h[o] + P[fc1_b + o], 0.0f);
    float* y = A + act_y;
    if (m->n_conv == 0)
      gemm_chunked(P + fc2_w, h, y, out_dim, m->fc_hidden);
    else
      gemm(P + fc2_w, h, y, out_dim, m->fc_hidden, 1, false);
    for (int o = 0; o < out_dim; ++o) y[o] += P[fc2_b + o];
    std::copy(y, y + out_dim, out);
  }
};

// cnn.cpp:388-402 (strict '>' argmax; fp64 FMA de-normalisation; llround).
uint32_t decode_head(const float* logits, int n, float r, double mu, double sigma) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (logits[i] > logits[best]) best = i;
  if (best < n - 1) return static_cast<uint32_t>(best);
  const double z = std::min(std::fma(static_cast<double>(r), sigma, mu), 22.0);
  const double raw = std::max(0.0, std::expm1(z));
  const long long v = std::llround(std::min(raw, 4.0e9));
  return static_cast<uint32_t>(std::min<long long>(v, 0xffffffffLL));
}

// cnn.cpp:406-417
void decode_triple(const port_model* m, const float* y, bool is_store, uint32_t* t) {
  const double* lm = m->norm + 100;
  const double* ls = m->norm + 103;
  const float* f = y + 3;
  const float* e = f + m->class_fetch;
  const float* s = e + m->class_exec;
  t[0] = decode_head(f, m->class_fetch, y[0], lm[0], ls[0]);
  t[1] = std::max<uint32_t>(1u, decode_head(e, m->class_exec, y[1], lm[1], ls[1]));
  t[2] = is_store ? decode_head(s, m->class_store, y[2], lm[2], ls[2]) : 0u;
}

// ---------------------------------------------------------------------------
// Feature helpers (dataset.cpp:47-75)
// ---------------------------------------------------------------------------
inline bool is_store_op(const port_trace* t, uint64_t i) { return t->op[i * 13 + kOpIsStore] != 0; }
inline bool is_mem_op(const port_trace* t, uint64_t i) {
  return t->op[i * 13 + kOpIsLoad] != 0 || t->op[i * 13 + kOpIsStore] != 0;
}

void dep_flags(const port_trace* t, uint64_t tgt, uint64_t ctx, uint32_t line, uint32_t page,
               int32_t* f) {
  const uint64_t pa = t->pc[tgt], pb = t->pc[ctx];
  f[0] = (pa / line) == (pb / line);
  f[1] = f[2] = f[3] = 0;
  if (is_mem_op(t, tgt) && is_mem_op(t, ctx)) {
    const uint64_t da = t->data_addr[tgt], db = t->data_addr[ctx];
    f[1] = da == db;
    f[2] = (da / line) == (db / line);
    f[3] = (da / page) == (db / page);
  }
  f[4] = (pa / page) == (pb / page);
}

// 41 static slots of one instruction, then residence/execution/store/flags/0.
void raw_column(const port_trace* t, uint64_t i, int64_t res, int64_t exe, int64_t sto,
                const int32_t* flags, int32_t* out) {
  int k = 0;
  for (int j = 0; j < 13; ++j) out[k++] = t->op[i * 13 + j];
  for (int j = 0; j < 8; ++j) out[k++] = t->src[i * 8 + j];
  for (int j = 0; j < 6; ++j) out[k++] = t->dst[i * 6 + j];
  for (int j = 0; j < 14; ++j) out[k++] = t->hist[i * 14 + j];
  out[k++] = static_cast<int32_t>(res);
  out[k++] = static_cast<int32_t>(exe);
  out[k++] = static_cast<int32_t>(sto);
  for (int j = 0; j < 5; ++j) out[k++] = flags ? flags[j] : 0;
  out[k++] = 0;
}

// ---------------------------------------------------------------------------
// One machine (restates simcore.cpp:10-174 with explicit residence counters)
// ---------------------------------------------------------------------------
struct Entry {
  uint32_t local, residence, execution, store;
  bool is_store;
};

struct Machine {
  const port_trace* t;
  uint64_t begin, len, warm;   // simulated global range [begin, begin+len); first `warm` are warm-up
  int max_context;
  uint32_t bw, line, page;
  bool per_cycle, record, count_drain;
  std::deque<Entry> proc, wq;
  uint64_t cur = 0, sum_fetch = 0, overflow = 0, drain_cyc = 0, pos = 0;
  uint64_t base_cur = 0, base_overflow = 0;
  std::vector<uint32_t> fetch;

  bool left() const { return pos < len; }

  size_t retire(uint64_t budget) {  // simcore.cpp:68-84
    size_t ev = 0;
    while (budget > 0 && !proc.empty()) {
      const Entry h = proc.front();
      if (h.residence < h.execution) break;
      if (h.is_store) wq.push_back(h);
      proc.pop_front();
      --budget;
      ++ev;
    }
    while (!wq.empty() && wq.front().residence >= wq.front().store) {
      wq.pop_front();
      ++ev;
    }
    return ev;
  }

  size_t advance(uint64_t cycles, uint64_t budget, uint64_t* counter) {  // simcore.cpp:86-93
    if (cycles == 0) return 0;
    cur += cycles;
    if (counter) *counter += cycles;
    for (Entry& e : proc) e.residence += static_cast<uint32_t>(cycles);
    for (Entry& e : wq) e.residence += static_cast<uint32_t>(cycles);
    return retire(budget);
  }

  uint64_t ready_gap() const {  // simcore.cpp:95-110
    uint64_t best = std::numeric_limits<uint64_t>::max();
    if (!proc.empty()) {
      const Entry& h = proc.front();
      best = std::min<uint64_t>(best, h.execution > h.residence ? h.execution - h.residence : 1);
    }
    if (!wq.empty()) {
      const Entry& h = wq.front();
      best = std::min<uint64_t>(best, h.store > h.residence ? h.store - h.residence : 1);
    }
    return best == std::numeric_limits<uint64_t>::max() ? 1 : std::max<uint64_t>(1, best);
  }

  // simcore.cpp:25-66: column 0 = target, then proc newest->oldest, then
  // write queue newest->oldest, <= max_context columns, rest exactly 0.
  void build_input(const double* mean, const double* sd, float* dst) const {
    const size_t width = static_cast<size_t>(kSlots) * (max_context + 1);
    std::fill(dst, dst + width, 0.0f);
    const uint64_t tgt = begin + pos;
    int32_t raw[kSlots];
    auto emit = [&](int col) {
      float* d = dst + static_cast<size_t>(col) * kSlots;
      for (int k = 0; k < kSlots; ++k) {
        const double z = (static_cast<double>(raw[k]) - mean[k]) / sd[k];
        d[k] = static_cast<float>(std::clamp(z, -10.0, 10.0));
      }
    };
    raw_column(t, tgt, 0, 0, 0, nullptr, raw);
    emit(0);
    int col = 1;
    const int max_cols = max_context + 1;
    int32_t f[5];
    for (auto it = proc.rbegin(); it != proc.rend() && col < max_cols; ++it) {
      dep_flags(t, tgt, begin + it->local, line, page, f);
      raw_column(t, begin + it->local, it->residence, it->execution, it->store, f, raw);
      emit(col++);
    }
    for (auto it = wq.rbegin(); it != wq.rend() && col < max_cols; ++it) {
      dep_flags(t, tgt, begin + it->local, line, page, f);
      raw_column(t, begin + it->local, it->residence, it->execution, it->store, f, raw);
      emit(col++);
    }
  }

  void apply(const uint32_t* trip) {  // simcore.cpp:112-150
    const uint32_t F = trip[0];
    if (F > 0) {
      if (per_cycle) {
        for (uint32_t c = 0; c < F; ++c) advance(1, bw, nullptr);
      } else {
        advance(F, static_cast<uint64_t>(bw) * F, nullptr);
      }
    }
    while (proc.size() >= static_cast<size_t>(max_context)) {
      const size_t before = proc.size();
      const Entry& h = proc.front();
      const uint64_t gap = h.execution > h.residence ? h.execution - h.residence : 1;
      advance(gap, bw, &overflow);
      if (proc.size() >= before)
        throw PortError("processor queue stalled without progress at tick " + std::to_string(cur));
    }
    proc.push_back(Entry{static_cast<uint32_t>(pos), 0, trip[1], trip[2], is_store_op(t, begin + pos)});
    if (pos >= warm) {
      sum_fetch += F;
      if (record) fetch.push_back(F);
    }
    ++pos;
    if (pos == warm) {  // warm-up extension: counting starts here
      base_cur = cur;
      base_overflow = overflow;
    }
  }

  void drain() {  // simcore.cpp:152-159
    if (!count_drain) return;
    while (!proc.empty() || !wq.empty()) {
      if (advance(ready_gap(), bw, &drain_cyc) == 0)
        throw PortError("drain made no progress at tick " + std::to_string(cur));
    }
  }

  void result(port_sub* r) const {  // simcore.cpp:161-174
    r->instructions = len - warm;
    r->total_cycles = cur - base_cur;
    r->sum_fetch = sum_fetch;
    r->delta = r->total_cycles - sum_fetch;
    r->drain_cycles = drain_cyc;
    r->overflow_stall_cycles = overflow - base_overflow;
    r->empty = (len - warm) == 0;
  }
};

void put_err(char* err, int n, const char* msg) {
  if (err && n > 0) {
    std::strncpy(err, msg, static_cast<size_t>(n) - 1);
    err[n - 1] = 0;
  }
}

std::vector<uint64_t> partition_starts(uint64_t n, uint64_t k) {  // parallel.cpp:9-24
  if (k < 1 || k > std::max<uint64_t>(n, 1))
    throw PortError("sub-trace count " + std::to_string(k) + " out of range for trace of " +
                    std::to_string(n));
  std::vector<uint64_t> s;
  const uint64_t base = n / k, rem = n % k;
  uint64_t at = 0;
  for (uint64_t i = 0; i < k; ++i) {
    s.push_back(at);
    at += base + (i < rem ? 1 : 0);
  }
  return s;
}

// xoshiro256** seeded by splitmix64 (common.hpp:18-67), for init_weights.
uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s) w = x = mix64(x);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t out = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
  }
  float symmetric(float a) {
    const double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
    return static_cast<float>((2.0 * u - 1.0) * a);
  }
};

}  // namespace

extern "C" {

int port_decode(const port_model* m, const float* outputs, uint64_t n, const uint8_t* is_store,
                uint32_t* triples) {
  const int od = 3 + m->class_fetch + m->class_exec + m->class_store;
  for (uint64_t i = 0; i < n; ++i) decode_triple(m, outputs + i * od, is_store[i] != 0, triples + 3 * i);
  return 0;
}

int port_partition(uint64_t n, uint64_t k, uint64_t* starts, char* err, int errlen) {
  try {
    const auto s = partition_starts(n, k);
    std::copy(s.begin(), s.end(), starts);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

uint64_t port_param_count(const port_model* m) { return Net(m).n_params; }

uint64_t port_model_flops(const port_model* m) {  // cnn.cpp:319-333 (multiplications)
  uint64_t mults = 0;
  int cin = m->input_channels, len = m->sequence_length;
  for (int l = 0; l < m->n_conv; ++l) {
    len /= 2;
    const uint64_t one = static_cast<uint64_t>(m->conv[l]) * len * (2 * cin);
    mults += m->residual ? 2 * one : one;
    cin = m->conv[l];
  }
  const Net net(m);
  mults += static_cast<uint64_t>(m->fc_hidden) * net.flat;
  mults += static_cast<uint64_t>(net.out_dim) * m->fc_hidden;
  return mults;
}

// cnn.cpp:335-352: Rng(splitmix64(seed) ^ 0xC44), U(+-1/sqrt(cols)) per
// tensor in table order (w, b, [p] per conv; fc1.w, fc1.b, fc2.w, fc2.b).
int port_init_weights(port_model* m, uint64_t seed, float* out, char* err, int errlen) {
  try {
    const Net net(m);
    Xoshiro rng(mix64(seed) ^ 0xC44u);
    auto fill = [&](size_t off, size_t count, size_t cols) {
      const float bound = 1.0f / std::sqrt(static_cast<float>(std::max<size_t>(1, cols)));
      for (size_t i = 0; i < count; ++i) out[off + i] = rng.symmetric(bound);
    };
    int cin = m->input_channels;
    for (int l = 0; l < m->n_conv; ++l) {
      const size_t cout = m->conv[l];
      fill(net.w[l], cout * 2 * cin, 2 * cin);
      fill(net.b[l], cout, 1);
      if (m->residual) fill(net.p[l], cout * 2 * cin, 2 * cin);
      cin = m->conv[l];
    }
    fill(net.fc1_w, static_cast<size_t>(m->fc_hidden) * net.flat, net.flat);
    fill(net.fc1_b, m->fc_hidden, 1);
    fill(net.fc2_w, static_cast<size_t>(net.out_dim) * m->fc_hidden, m->fc_hidden);
    fill(net.fc2_b, net.out_dim, 1);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

int port_forward(const port_model* m, const float* inputs, uint64_t n, const uint8_t* is_store,
                 float* outputs, uint32_t* triples, char* err, int errlen) {
  try {
    const Net net(m);
    const size_t width = net.width();
#pragma omp parallel
    {
      std::vector<float> act;
      std::vector<float> y(net.out_dim);
#pragma omp for schedule(static)
      for (int64_t i = 0; i < static_cast<int64_t>(n); ++i) {
        net.forward(inputs + i * width, y.data(), act);
        if (outputs) std::copy(y.begin(), y.end(), outputs + i * net.out_dim);
        if (triples) decode_triple(m, y.data(), is_store[i] != 0, triples + 3 * i);
      }
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

int port_simulate(const port_trace* t, const port_model* m, const port_config* c, port_sub* subs,
                  uint64_t sub_cap, uint32_t* predicted_fetch, uint64_t* totals, port_capture* cap,
                  char* err, int errlen) {
  try {
#ifdef _OPENMP
    if (c->threads > 0) omp_set_num_threads(c->threads);
#endif
    const uint64_t n = t->n;
    const bool truth = c->oracle || c->truth_with_inputs;
    const bool needs_input = !c->oracle;
    if (!truth && !m) throw PortError("simulate requires a model or oracle mode");
    if (truth && !t->truth) throw PortError("oracle mode requires truth latencies");
    const int mc = c->max_context > 0 ? c->max_context : (m ? m->max_context : 110);
    if (!truth && mc != m->max_context) throw PortError("max_context differs from the model's");

    // parallel.cpp:28-40
    uint64_t k = c->k;
    if (c->sequential) {
      k = 1;
    } else {
      if (c->subtrace_size > 0) {
        const uint64_t derived = n == 0 ? 1 : (n + c->subtrace_size - 1) / c->subtrace_size;
        if (k == 0)
          k = derived;
        else if (k != derived)
          throw PortError("inconsistent partition: k=" + std::to_string(k) + " but subtrace size " +
                          std::to_string(c->subtrace_size) + " implies k=" + std::to_string(derived));
      }
      if (k == 0) k = 1;
      if (c->batch_max == 0) throw PortError("batch_max must be >= 1");
    }
    // simcore.cpp:13-18
    if (mc < 1) throw PortError("max_context must be >= 1");
    if (c->retire_bandwidth < 1) throw PortError("retire_bandwidth must be >= 1");
    if (needs_input && !m) throw PortError("predictor requires inputs but provides no normalization stats");

    if (n == 0 && !c->sequential) {  // parallel.cpp:44-50
      if (sub_cap < 1) throw PortError("sub_cap too small");
      subs[0] = port_sub{0, 0, 0, 0, 0, 0, 1};
      totals[0] = 1;
      totals[1] = 0;
      totals[2] = 0;
      return 0;
    }
    const std::vector<uint64_t> starts = c->sequential ? std::vector<uint64_t>{0} : partition_starts(n, k);
    if (k > sub_cap) throw PortError("sub_cap too small");

    std::vector<Machine> cores(k);
    for (uint64_t i = 0; i < k; ++i) {
      const uint64_t s = starts[i];
      const uint64_t e = i + 1 < k ? starts[i + 1] : n;
      const uint64_t w = std::min<uint64_t>(c->warmup, s);  // warm-up extension
      Machine& mm = cores[i];
      mm.t = t;
      mm.begin = s - w;
      mm.len = e - s + w;
      mm.warm = w;
      mm.max_context = mc;
      mm.bw = c->retire_bandwidth;
      mm.line = c->line_size;
      mm.page = c->page_size;
      mm.per_cycle = c->per_cycle_advance != 0;
      mm.record = c->record_fetch != 0;
      mm.count_drain = !(c->drain_trim && i + 1 < k);  // drain-trim extension
    }

    std::unique_ptr<Net> net;
    if (m && !c->oracle) net = std::make_unique<Net>(m);
    const size_t width = static_cast<size_t>(kSlots) * (mc + 1);
    const int od = net ? net->out_dim : 0;
    const double* mean = m ? m->norm : nullptr;
    const double* sd = m ? m->norm + 50 : nullptr;

    std::vector<uint64_t> active;
    std::vector<float> inputs, outs;
    std::vector<uint32_t> trip;
    uint64_t produced = 0;
    uint32_t round = 0;
    for (;; ++round) {  // parallel.cpp:63-81
      active.clear();
      for (uint64_t i = 0; i < k; ++i)
        if (cores[i].left()) active.push_back(i);
      if (active.empty()) break;
      const size_t B = active.size();
      trip.assign(3 * B, 0);
      if (needs_input) {
        inputs.resize(B * width);
        for (size_t j = 0; j < B; ++j) cores[active[j]].build_input(mean, sd, inputs.data() + j * width);
      }
      if (truth) {
        for (size_t j = 0; j < B; ++j) {
          const Machine& mm = cores[active[j]];
          const uint32_t* tr = t->truth + 3 * (mm.begin + mm.pos);
          std::copy(tr, tr + 3, trip.data() + 3 * j);
        }
      } else {
        outs.resize(B * od);
#pragma omp parallel
        {
          std::vector<float> act;
#pragma omp for schedule(static)
          for (int64_t j = 0; j < static_cast<int64_t>(B); ++j) {
            net->forward(inputs.data() + j * width, outs.data() + j * od, act);
            const Machine& mm = cores[active[j]];
            decode_triple(m, outs.data() + j * od, is_store_op(t, mm.begin + mm.pos), trip.data() + 3 * j);
          }
        }
      }
      if (cap) {
        for (size_t j = 0; j < B; ++j, ++produced) {
          if (produced >= cap->cap) continue;
          const Machine& mm = cores[active[j]];
          const uint64_t r = produced;
          if (cap->inputs && needs_input)
            std::copy(inputs.begin() + j * width, inputs.begin() + (j + 1) * width, cap->inputs + r * width);
          if (cap->outputs && od)
            std::copy(outs.begin() + j * od, outs.begin() + (j + 1) * od, cap->outputs + r * od);
          if (cap->index) cap->index[r] = mm.begin + mm.pos;
          if (cap->is_store) cap->is_store[r] = is_store_op(t, mm.begin + mm.pos);
          if (cap->triples) std::copy(trip.begin() + 3 * j, trip.begin() + 3 * j + 3, cap->triples + 3 * r);
          if (cap->round) cap->round[r] = round;
        }
      }
      for (size_t j = 0; j < B; ++j) {
        Machine& mm = cores[active[j]];
        mm.apply(trip.data() + 3 * j);
        if (!mm.left()) mm.drain();
      }
    }
    if (cap) cap->count = produced;

    uint64_t total = 0, off = 0;
    for (uint64_t i = 0; i < k; ++i) {
      cores[i].result(&subs[i]);
      total += subs[i].total_cycles;
      if (predicted_fetch && c->record_fetch) {
        std::copy(cores[i].fetch.begin(), cores[i].fetch.end(), predicted_fetch + off);
        off += cores[i].fetch.size();
      }
    }
    totals[0] = k;
    totals[1] = total;
    totals[2] = n;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

}  // extern "C"
