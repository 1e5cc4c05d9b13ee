// TEST INFRASTRUCTURE ONLY — part of the CPU oracle, never linked into the product.
//
// Eigen-free restatement of the inference half of the reference's
// proj/src/cnn.cpp.  The reference forward runs its GEMMs through Eigen
// (cnn.cpp:8, 99-124); Eigen3 is not installed in this image, so cnn.cpp does
// not compile here.  This file provides the same symbols (declared in the
// reference header proj/include/ilsim/cnn.hpp) so the reference's own
// predictor.cpp / simcore.cpp / parallel.cpp can be linked unmodified
// (oracle/Makefile) and so the oracle port can share one forward.
//
// What is restated, and from where:
//   parameter / activation offsets   cnn.cpp:44-86   (make_offsets)
//   forward order GEMM->bias->ReLU   cnn.cpp:90-125  (forward_core), residual P*in before bias
//   padding 111 -> 128 columns       cnn.cpp:219-225 (pad_input)
//   config checks / hash / presets   cnn.cpp:229-281
//   tensor table, flops, init        cnn.cpp:293-352
//   output split                     cnn.cpp:354-368
//   hybrid decode                    cnn.cpp:388-417
//   ILMD model files                 cnn.cpp:635-697
// Training (loss/backward/Adam/eval) is off the simulate path and not restated.
//
// Arithmetic note: each GEMM is accumulated k-ascending per output with fused
// multiply-add (the reference's -march=native build contracts the same
// products); Eigen's blocked order is unknowable without Eigen, so forward
// parity with the reference binary is pinned to the reference's own tolerance
// (test_cnn.cpp:155-168, 1e-6 relative vs a double-precision naive forward).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "ilsim/cnn.hpp"
#include "ilsim/common.hpp"

namespace ilsim {

namespace {

struct Layout {
  std::vector<size_t> w, b, p;  // per conv layer: weight, bias, residual projection
  size_t fc1_w = 0, fc1_b = 0, fc2_w = 0, fc2_b = 0, n_params = 0;
  std::vector<size_t> act;      // activation offsets: input then each conv output
  size_t act_h = 0, act_y = 0, act_n = 0;
};

// cnn.cpp:44-86
Layout layout_of(const CnnConfig& c) {
  Layout L;
  size_t off = 0;
  int cin = c.input_channels;
  for (int cout : c.conv_channels) {
    const size_t taps = static_cast<size_t>(cout) * 2 * cin;
    L.w.push_back(off);
    off += taps;
    L.b.push_back(off);
    off += cout;
    if (c.residual_blocks) {
      L.p.push_back(off);
      off += taps;
    }
    cin = cout;
  }
  L.fc1_w = off;
  off += static_cast<size_t>(c.fc_hidden) * c.flat_dim();
  L.fc1_b = off;
  off += c.fc_hidden;
  L.fc2_w = off;
  off += static_cast<size_t>(c.output_dim()) * c.fc_hidden;
  L.fc2_b = off;
  off += c.output_dim();
  L.n_params = off;

  size_t a = 0;
  int len = c.sequence_length;
  L.act.push_back(a);
  a += static_cast<size_t>(c.input_channels) * len;
  for (int cout : c.conv_channels) {
    len >>= 1;
    L.act.push_back(a);
    a += static_cast<size_t>(cout) * len;
  }
  L.act_h = a;
  a += c.fc_hidden;
  L.act_y = a;
  a += c.output_dim();
  L.act_n = a;
  return L;
}

// y[rows x cols] (+)= W[rows x inner] * x[inner x cols], all column-major.
// k-ascending accumulation per output element.
void gemm_cm(const float* W, const float* x, float* y, int rows, int inner, int cols,
             bool accumulate) {
  for (int j = 0; j < cols; ++j) {
    float* yj = y + static_cast<size_t>(j) * rows;
    if (!accumulate) std::fill(yj, yj + rows, 0.0f);
    const float* xj = x + static_cast<size_t>(j) * inner;
    for (int k = 0; k < inner; ++k) {
      const float a = xj[k];
      const float* wk = W + static_cast<size_t>(k) * rows;
      for (int o = 0; o < rows; ++o) yj[o] = std::fma(wk[o], a, yj[o]);
    }
  }
}

// cnn.cpp:90-125: per layer out = W*in (+P*in), += bias, ReLU; then FC1+ReLU, FC2.
void run_forward(const CnnConfig& c, const Layout& L, const float* prm, float* act) {
  int cin = c.input_channels;
  int len = c.sequence_length;
  for (int l = 0; l < c.conv_layers(); ++l) {
    const int cout = c.conv_channels[l];
    const int olen = len / 2;
    const float* in = act + L.act[l];  // [2*cin x olen] column-major: k2/s2 windows are contiguous
    float* out = act + L.act[l + 1];   // [cout x olen]
    gemm_cm(prm + L.w[l], in, out, cout, 2 * cin, olen, false);
    if (c.residual_blocks) gemm_cm(prm + L.p[l], in, out, cout, 2 * cin, olen, true);
    const float* b = prm + L.b[l];
    for (int j = 0; j < olen; ++j)
      for (int o = 0; o < cout; ++o) {
        float& v = out[static_cast<size_t>(j) * cout + o];
        v = std::max(v + b[o], 0.0f);
      }
    cin = cout;
    len = olen;
  }
  const float* flat = act + L.act[c.conv_layers()];
  float* h = act + L.act_h;
  gemm_cm(prm + L.fc1_w, flat, h, c.fc_hidden, c.flat_dim(), 1, false);
  for (int o = 0; o < c.fc_hidden; ++o) h[o] = std::max(h[o] + prm[L.fc1_b + o], 0.0f);
  float* y = act + L.act_y;
  gemm_cm(prm + L.fc2_w, h, y, c.output_dim(), c.fc_hidden, 1, false);
  for (int o = 0; o < c.output_dim(); ++o) y[o] += prm[L.fc2_b + o];
}

// cnn.cpp:388-393: strict '>' keeps the first maximum; NaN never wins.
int first_argmax(const float* v, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

// cnn.cpp:395-402.  r*sigma+mu is one fp64 FMA under the reference's
// -march=native build (GCC contracts it); std::fma makes that explicit.
uint32_t decode_one(const float* logits, int n, float r, double mu, double sigma) {
  const int cls = first_argmax(logits, n);
  if (cls < n - 1) return static_cast<uint32_t>(cls);
  const double z = std::min(std::fma(static_cast<double>(r), sigma, mu), 22.0);
  const double raw = std::max(0.0, std::expm1(z));
  const long long v = std::llround(std::min(raw, 4.0e9));
  return static_cast<uint32_t>(std::min<long long>(v, 0xffffffffLL));
}

}  // namespace

// ---- CnnConfig (cnn.cpp:229-281) -------------------------------------------

void CnnConfig::validate_or_throw() const {
  if (input_channels < 1) throw Error("input_channels must be >= 1");
  if (max_context < 0) throw Error("max_context must be >= 0");
  if (conv_channels.empty()) throw Error("at least one conv layer required");
  for (int ch : conv_channels)
    if (ch < 1) throw Error("conv channel counts must be >= 1");
  if (sequence_length < max_context + 1) throw Error("sequence_length smaller than max_context + 1");
  if (sequence_length % (1 << conv_layers()) != 0)
    throw Error("sequence_length must be divisible by 2^conv_layers");
  if (fc_hidden < 1) throw Error("fc_hidden must be >= 1");
  if (class_fetch < 2 || class_exec < 2 || class_store < 2)
    throw Error("class counts must be >= 2");
}

uint64_t CnnConfig::hash() const {
  uint64_t h = 0xcbf29ce484222325ULL;
  auto feed = [&h](uint64_t v) { h = fnv1a64(&v, sizeof v, h); };
  feed(static_cast<uint64_t>(input_channels));
  feed(static_cast<uint64_t>(max_context));
  feed(static_cast<uint64_t>(sequence_length));
  for (int ch : conv_channels) feed(static_cast<uint64_t>(ch));
  feed(static_cast<uint64_t>(fc_hidden));
  feed(static_cast<uint64_t>(class_fetch));
  feed(static_cast<uint64_t>(class_exec));
  feed(static_cast<uint64_t>(class_store));
  feed(residual_blocks ? 1u : 0u);
  return h;
}

CnnConfig CnnConfig::preset_c3(int max_context) {
  CnnConfig c;
  c.max_context = max_context;
  c.conv_channels = {64, 64, 64};
  c.fc_hidden = 256;
  int seq = 1;
  while (seq < max_context + 1) seq *= 2;
  c.sequence_length = std::max(seq, 1 << c.conv_layers());
  return c;
}

CnnConfig CnnConfig::tiny(int channels, int seq) {
  CnnConfig c;
  c.input_channels = channels;
  c.max_context = seq - 1;
  c.sequence_length = seq;
  c.conv_channels = {6, 6};
  c.fc_hidden = 8;
  return c;
}

// ---- tensor table / counts / init (cnn.cpp:293-352) ------------------------

std::vector<TensorShape> tensor_table(const CnnConfig& c) {
  c.validate_or_throw();
  const Layout L = layout_of(c);
  std::vector<TensorShape> t;
  int cin = c.input_channels;
  for (int l = 0; l < c.conv_layers(); ++l) {
    const size_t cout = static_cast<size_t>(c.conv_channels[l]);
    const std::string pre = "conv" + std::to_string(l);
    t.push_back({pre + ".w", L.w[l], cout, static_cast<size_t>(2 * cin)});
    t.push_back({pre + ".b", L.b[l], cout, 1});
    if (c.residual_blocks) t.push_back({pre + ".p", L.p[l], cout, static_cast<size_t>(2 * cin)});
    cin = c.conv_channels[l];
  }
  t.push_back({"fc1.w", L.fc1_w, static_cast<size_t>(c.fc_hidden), static_cast<size_t>(c.flat_dim())});
  t.push_back({"fc1.b", L.fc1_b, static_cast<size_t>(c.fc_hidden), 1});
  t.push_back({"fc2.w", L.fc2_w, static_cast<size_t>(c.output_dim()), static_cast<size_t>(c.fc_hidden)});
  t.push_back({"fc2.b", L.fc2_b, static_cast<size_t>(c.output_dim()), 1});
  return t;
}

size_t param_count(const CnnConfig& c) { return layout_of(c).n_params; }

uint64_t model_flops(const CnnConfig& c) {
  uint64_t mults = 0;
  int cin = c.input_channels;
  int len = c.sequence_length;
  for (int cout : c.conv_channels) {
    len /= 2;
    const uint64_t one = static_cast<uint64_t>(cout) * len * (2 * cin);
    mults += c.residual_blocks ? 2 * one : one;
    cin = cout;
  }
  mults += static_cast<uint64_t>(c.fc_hidden) * c.flat_dim();
  mults += static_cast<uint64_t>(c.output_dim()) * c.fc_hidden;
  return mults;
}

ModelWeights init_weights(const CnnConfig& c, const NormStats& norm, uint64_t seed) {
  c.validate_or_throw();
  ModelWeights w;
  w.config = c;
  w.norm = norm;
  const size_t n = param_count(c);
  w.params.assign(n, 0.0f);
  w.adam_m.assign(n, 0.0f);
  w.adam_v.assign(n, 0.0f);
  Rng rng(splitmix64(seed) ^ 0xC44u);
  for (const TensorShape& t : tensor_table(c)) {
    // U(+-1/sqrt(cols)); bias tensors have cols == 1 and so draw from U(+-1).
    const float bound = 1.0f / std::sqrt(static_cast<float>(std::max<size_t>(1, t.cols)));
    for (size_t i = 0; i < t.count(); ++i) w.params[t.offset + i] = rng.next_symmetric(bound);
  }
  return w;
}

// ---- forward + decode (cnn.cpp:219-225, 354-368, 388-417) ------------------

PredictionOutput forward(const ModelWeights& w, const float* input, CnnWorkspace& ws) {
  const CnnConfig& c = w.config;
  const Layout L = layout_of(c);
  ws.act.resize(L.act_n);
  const size_t real = static_cast<size_t>(c.input_channels) * (c.max_context + 1);
  const size_t padded = static_cast<size_t>(c.input_channels) * c.sequence_length;
  std::copy(input, input + real, ws.act.begin());
  std::fill(ws.act.begin() + real, ws.act.begin() + padded, 0.0f);
  run_forward(c, L, w.params.data(), ws.act.data());
  const float* y = ws.act.data() + L.act_y;
  PredictionOutput out;
  for (int i = 0; i < 3; ++i) out.regression[i] = y[i];
  const float* f = y + 3;
  const float* e = f + c.class_fetch;
  const float* s = e + c.class_exec;
  out.fetch_logits.assign(f, f + c.class_fetch);
  out.exec_logits.assign(e, e + c.class_exec);
  out.store_logits.assign(s, s + c.class_store);
  return out;
}

LatencyTriple decode_hybrid(const PredictionOutput& out, const NormStats& norm, bool target_is_store) {
  LatencyTriple t;
  t.fetch = decode_one(out.fetch_logits.data(), static_cast<int>(out.fetch_logits.size()),
                       out.regression[0], norm.label_mean[0], norm.label_stdev[0]);
  t.execution = std::max<uint32_t>(
      1u, decode_one(out.exec_logits.data(), static_cast<int>(out.exec_logits.size()),
                     out.regression[1], norm.label_mean[1], norm.label_stdev[1]));
  t.store = target_is_store
                ? decode_one(out.store_logits.data(), static_cast<int>(out.store_logits.size()),
                             out.regression[2], norm.label_mean[2], norm.label_stdev[2])
                : 0u;
  return t;
}

// ---- ILMD model files (cnn.cpp:635-697) ------------------------------------

namespace {
const char kIlmd[4] = {'I', 'L', 'M', 'D'};
}

void save_model(const std::string& path, const ModelWeights& w) {
  BinaryWriter o(path);
  o.write_bytes(kIlmd, 4);
  o.write<uint32_t>(1);
  o.write<uint64_t>(w.config.hash());
  o.write<uint32_t>(w.config.input_channels);
  o.write<uint32_t>(w.config.max_context);
  o.write<uint32_t>(w.config.sequence_length);
  o.write<uint32_t>(static_cast<uint32_t>(w.config.conv_channels.size()));
  for (int ch : w.config.conv_channels) o.write<uint32_t>(ch);
  o.write<uint32_t>(w.config.fc_hidden);
  o.write<uint32_t>(w.config.class_fetch);
  o.write<uint32_t>(w.config.class_exec);
  o.write<uint32_t>(w.config.class_store);
  o.write<uint8_t>(w.config.residual_blocks ? 1 : 0);
  for (double v : w.norm.mean) o.write_f64(v);
  for (double v : w.norm.stdev) o.write_f64(v);
  for (double v : w.norm.label_mean) o.write_f64(v);
  for (double v : w.norm.label_stdev) o.write_f64(v);
  o.write<int64_t>(w.adam_step);
  o.write<uint64_t>(w.params.size());
  for (float v : w.params) o.write_f32(v);
  for (float v : w.adam_m) o.write_f32(v);
  for (float v : w.adam_v) o.write_f32(v);
  o.close();
}

ModelWeights load_model(const std::string& path) {
  BinaryReader in(path);
  char magic[4];
  in.read_bytes(magic, 4);
  if (std::memcmp(magic, kIlmd, 4) != 0) throw Error("bad model magic in " + path);
  if (in.read<uint32_t>() != 1) throw Error("unsupported model version");
  const uint64_t want_hash = in.read<uint64_t>();
  ModelWeights w;
  CnnConfig& c = w.config;
  c.input_channels = static_cast<int>(in.read<uint32_t>());
  c.max_context = static_cast<int>(in.read<uint32_t>());
  c.sequence_length = static_cast<int>(in.read<uint32_t>());
  c.conv_channels.resize(in.read<uint32_t>());
  for (int& ch : c.conv_channels) ch = static_cast<int>(in.read<uint32_t>());
  c.fc_hidden = static_cast<int>(in.read<uint32_t>());
  c.class_fetch = static_cast<int>(in.read<uint32_t>());
  c.class_exec = static_cast<int>(in.read<uint32_t>());
  c.class_store = static_cast<int>(in.read<uint32_t>());
  c.residual_blocks = in.read<uint8_t>() != 0;
  if (c.hash() != want_hash) throw Error("model config hash mismatch in " + path);
  for (double& v : w.norm.mean) v = in.read_f64();
  for (double& v : w.norm.stdev) v = in.read_f64();
  for (double& v : w.norm.label_mean) v = in.read_f64();
  for (double& v : w.norm.label_stdev) v = in.read_f64();
  w.adam_step = in.read<int64_t>();
  const uint64_t n = in.read<uint64_t>();
  if (n != param_count(c)) throw Error("model parameter count mismatch in " + path);
  w.params.resize(n);
  w.adam_m.resize(n);
  w.adam_v.resize(n);
  for (float& v : w.params) v = in.read_f32();
  for (float& v : w.adam_m) v = in.read_f32();
  for (float& v : w.adam_v) v = in.read_f32();
  return w;
}

}  // namespace ilsim
