// Model bookkeeping and the K2 forward dispatch.
#include <cmath>
#include <cstring>

#include "gemm.cuh"
#include "model.cuh"

namespace simnet {

ParamLayout param_layout(const ilsim_cnn_config& c) {  // cnn.cpp:44-86
  ParamLayout L;
  L.out_dim = 3 + c.class_fetch + c.class_exec + c.class_store;
  // n_conv == 0: the FC-only predictor (extension; PAPER.md:794 FC2), FC1 on
  // the unpadded input of 50 x (max_context + 1) slots
  L.flat = c.n_conv == 0 ? c.input_channels * (c.max_context + 1)
                         : c.conv[c.n_conv - 1] * (c.sequence_length >> c.n_conv);
  uint64_t off = 0;
  int cin = c.input_channels;
  for (int l = 0; l < c.n_conv; ++l) {
    const uint64_t taps = static_cast<uint64_t>(c.conv[l]) * 2 * cin;
    L.w.push_back(off);
    off += taps;
    L.b.push_back(off);
    off += c.conv[l];
    if (c.residual) {
      L.p.push_back(off);
      off += taps;
    }
    cin = c.conv[l];
  }
  L.fc1_w = off;
  off += static_cast<uint64_t>(c.fc_hidden) * L.flat;
  L.fc1_b = off;
  off += c.fc_hidden;
  L.fc2_w = off;
  off += static_cast<uint64_t>(L.out_dim) * c.fc_hidden;
  L.fc2_b = off;
  off += L.out_dim;
  L.total = off;
  return L;
}

// CnnConfig::validate_or_throw (cnn.cpp:229-243) + what the GPU path needs.
void validate_config(const ilsim_cnn_config& c) {
  if (c.input_channels < 1) throw ApiError("input_channels must be >= 1");
  if (c.max_context < 0) throw ApiError("max_context must be >= 0");
  if (c.n_conv < 0) throw ApiError("conv layer count must be >= 0");
  if (c.n_conv > 8) throw ApiError("at most 8 conv layers supported");
  for (int l = 0; l < c.n_conv; ++l)
    if (c.conv[l] < 1) throw ApiError("conv channel counts must be >= 1");
  if (c.sequence_length < c.max_context + 1) throw ApiError("sequence_length smaller than max_context + 1");
  if (c.sequence_length % (1 << c.n_conv) != 0)
    throw ApiError("sequence_length must be divisible by 2^conv_layers");
  if (c.fc_hidden < 1) throw ApiError("fc_hidden must be >= 1");
  if (c.class_fetch < 2 || c.class_exec < 2 || c.class_store < 2)
    throw ApiError("class counts must be >= 2");
  if (c.input_channels != 50) throw ApiError("the simulator's feature layout has 50 slots per column");
}

uint64_t param_count_of(const ilsim_cnn_config& c) { return param_layout(c).total; }
int output_dim_of(const ilsim_cnn_config& c) { return 3 + c.class_fetch + c.class_exec + c.class_store; }

uint64_t model_flops_of(const ilsim_cnn_config& c) {  // cnn.cpp:319-333 (multiplications)
  uint64_t mults = 0;
  int cin = c.input_channels, len = c.sequence_length;
  for (int l = 0; l < c.n_conv; ++l) {
    len /= 2;
    const uint64_t one = static_cast<uint64_t>(c.conv[l]) * len * (2 * cin);
    mults += c.residual ? 2 * one : one;
    cin = c.conv[l];
  }
  const ParamLayout L = param_layout(c);
  mults += static_cast<uint64_t>(c.fc_hidden) * L.flat;
  mults += static_cast<uint64_t>(L.out_dim) * c.fc_hidden;
  return mults;
}

namespace {
uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
}  // namespace

// init_weights (cnn.cpp:335-352): xoshiro256** seeded from
// splitmix64(seed) ^ 0xC44, U(+-1/sqrt(cols)) per tensor in table order.
void init_weights_into(const ilsim_cnn_config& c, uint64_t seed, float* out) {
  const ParamLayout L = param_layout(c);
  uint64_t s[4];
  uint64_t x = splitmix(seed) ^ 0xC44u;
  for (auto& w : s) w = x = splitmix(x);
  auto rotl = [](uint64_t v, int k) { return (v << k) | (v >> (64 - k)); };
  auto next = [&]() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  };
  auto fill = [&](uint64_t off, uint64_t count, uint64_t cols) {
    const float bound = 1.0f / std::sqrt(static_cast<float>(cols < 1 ? 1 : cols));
    for (uint64_t i = 0; i < count; ++i) {
      const double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
      out[off + i] = static_cast<float>((2.0 * u - 1.0) * bound);
    }
  };
  int cin = c.input_channels;
  for (int l = 0; l < c.n_conv; ++l) {
    const uint64_t cout = c.conv[l];
    fill(L.w[l], cout * 2 * cin, 2 * cin);
    fill(L.b[l], cout, 1);
    if (c.residual) fill(L.p[l], cout * 2 * cin, 2 * cin);
    cin = c.conv[l];
  }
  fill(L.fc1_w, static_cast<uint64_t>(c.fc_hidden) * L.flat, L.flat);
  fill(L.fc1_b, c.fc_hidden, 1);
  fill(L.fc2_w, static_cast<uint64_t>(L.out_dim) * c.fc_hidden, c.fc_hidden);
  fill(L.fc2_b, L.out_dim, 1);
}

bool split_input(const DevModel& m) { return m.tc != nullptr && tc_split_input(m.tc); }

DevModel::~DevModel() {
  if (tc) tc_model_destroy(tc);
}

void model_upload(DevModel& m, const ilsim_cnn_config& c, const float* params, int precision,
                  cudaStream_t s) {
  m.cfg = c;
  m.L = param_layout(c);
  m.params.need(m.L.total * sizeof(float));
  CUDA_OK(cudaMemcpyAsync(m.params.p, params, m.L.total * sizeof(float), cudaMemcpyHostToDevice, s));
  if (m.tc) {
    tc_model_destroy(m.tc);
    m.tc = nullptr;
  }
  if (precision != ILSIM_PREC_FP32) {
    m.tc = tc_model_create(m, params, precision, s);
    tc_calibrate(m, s);
  }
}

ForwardBuffers forward_buffers(const DevModel& m, uint64_t chunk, DevBuf& act, DevBuf& y) {
  const ilsim_cnn_config& c = m.cfg;
  ForwardBuffers fb{};
  uint64_t floats = 0;
  std::vector<uint64_t> off;
  int len = c.sequence_length;
  for (int l = 0; l < c.n_conv; ++l) {
    len /= 2;
    off.push_back(floats);
    floats += chunk * static_cast<uint64_t>(len) * c.conv[l];
    floats = (floats + 63) & ~63ull;
  }
  off.push_back(floats);
  floats += chunk * static_cast<uint64_t>(c.fc_hidden);
  floats = (floats + 63) & ~63ull;
  const uint64_t sk_off = floats;
  const bool sk = chunk <= kSgemvMaxM;  // sequential / tiny batches: split-K GEMV for the FC layers
  if (sk)
    floats += std::max(sgemm_splitk_floats(chunk, m.L.flat, c.fc_hidden),
                       sgemm_splitk_floats(chunk, c.fc_hidden, m.L.out_dim));
  float* base = static_cast<float*>(act.need(floats * sizeof(float)));
  for (size_t i = 0; i < off.size(); ++i) fb.act[i] = base + off[i];
  fb.splitk = sk ? base + sk_off : nullptr;
  fb.y_stride = static_cast<uint32_t>(m.L.out_dim);
  fb.y = static_cast<float*>(y.need(chunk * fb.y_stride * sizeof(float)));
  if (m.tc) tc_prepare(m, chunk);
  fb.act_esz = m.tc ? tc_act_bytes(m.tc) : 4u;
  fb.part_off = 0;
  return fb;
}

ForwardBuffers fb_slice(const DevModel& m, const ForwardBuffers& fb, uint64_t off) {
  const ilsim_cnn_config& c = m.cfg;
  ForwardBuffers s = fb;
  int len = c.sequence_length;
  for (int l = 0; l < c.n_conv; ++l) {
    len /= 2;
    const uint64_t bytes = off * static_cast<uint64_t>(len) * c.conv[l] * fb.act_esz;
    s.act[l] = reinterpret_cast<float*>(reinterpret_cast<char*>(fb.act[l]) + bytes);
  }
  s.act[c.n_conv] = fb.act[c.n_conv] + off * static_cast<uint64_t>(c.fc_hidden);
  s.y = fb.y + off * fb.y_stride;
  s.part_off = fb.part_off + off;
  if (off > 0) s.splitk = nullptr;  // one scratch: only the first slice may use it
  return s;
}

uint64_t forward_launch(const DevModel& m, int precision, const void* xv, uint32_t x_stride,
                        uint64_t samples, const ForwardBuffers& fb, cudaStream_t s, const DecodeParams* fuse,
                        bool* fused, uint64_t x_lo_off) {
  if (fused) *fused = false;
  if (precision != ILSIM_PREC_FP32) {
    if (fused) *fused = fuse != nullptr;
    return tc_forward(m, precision, xv, x_stride, samples, fb, s, fuse, x_lo_off);
  }
  const float* x = static_cast<const float*>(xv);
  const ilsim_cnn_config& c = m.cfg;
  const float* P = m.params.as<float>();
  uint64_t launches = 0;
  int cin = c.input_channels, len = c.sequence_length;
  const float* in = x;
  int valid = static_cast<int>(x_stride / (2 * cin));
  uint64_t sstride = x_stride;
  for (int l = 0; l < c.n_conv; ++l) {
    const int olen = len / 2, cout = c.conv[l];
    LayerGemm g{};
    g.a = in;
    g.m = samples * olen;
    g.rows_per_sample = olen;
    g.valid_rows = valid < olen ? valid : olen;
    g.kdim = 2 * cin;
    g.sample_stride = sstride;
    g.w = P + m.L.w[l];
    g.w2 = c.residual ? P + m.L.p[l] : nullptr;
    g.bias = P + m.L.b[l];
    g.c = fb.act[l];
    g.n = cout;
    g.ldc = cout;
    g.relu = 1;
    launch_sgemm(g, s);
    ++launches;
    in = fb.act[l];
    cin = cout;
    len = olen;
    valid = olen / 2;
    sstride = static_cast<uint64_t>(olen) * cout;
  }
  // accumulation order (gemm.cuh): the CNN models follow the reference's
  // restated forward (one chain per output); the FC-only predictor its own
  // 512-wide chunked definition (shared with the oracle port)
  const int fc_chunk = c.n_conv == 0 ? kSgemmChunk : 0;
  LayerGemm f1{};
  f1.chunk = fc_chunk;
  f1.a = in;
  f1.m = samples;
  f1.rows_per_sample = 1;
  f1.valid_rows = 1;
  f1.kdim = m.L.flat;
  f1.sample_stride = c.n_conv == 0 ? x_stride : m.L.flat;  // FC-only: FC1 reads the gathered rows
  f1.w = P + m.L.fc1_w;
  f1.bias = P + m.L.fc1_b;
  f1.c = fb.act[c.n_conv];
  f1.n = c.fc_hidden;
  f1.ldc = c.fc_hidden;
  f1.relu = 1;
  f1.splitk = fb.splitk;
  launch_sgemm(f1, s);
  LayerGemm f2{};
  f2.chunk = fc_chunk;
  f2.a = fb.act[c.n_conv];
  f2.m = samples;
  f2.rows_per_sample = 1;
  f2.valid_rows = 1;
  f2.kdim = c.fc_hidden;
  f2.sample_stride = c.fc_hidden;
  f2.w = P + m.L.fc2_w;
  f2.bias = P + m.L.fc2_b;
  f2.c = fb.y;
  f2.n = m.L.out_dim;
  f2.ldc = static_cast<int>(fb.y_stride);
  f2.relu = 0;
  f2.splitk = fb.splitk;
  launch_sgemm(f2, s);
  return launches + (sgemm_two_launches(f1) ? 2 : 1) + (sgemm_two_launches(f2) ? 2 : 1);
}

}  // namespace simnet
