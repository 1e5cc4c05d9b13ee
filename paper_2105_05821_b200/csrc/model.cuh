// Latency-predictor model on the device: CnnConfig checks and parameter
// layout (cnn.cpp:44-86, 229-352), weight upload in the operand layouts each
// K2 precision needs, and the per-chunk forward dispatch.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/ilsim_gpu.h"
#include "host_util.cuh"
#include "round_front.cuh"
#include "sim_kernels.cuh"

namespace simnet {

struct ParamLayout {
  std::vector<uint64_t> w, b, p;  // per conv layer (p: residual projection)
  uint64_t fc1_w = 0, fc1_b = 0, fc2_w = 0, fc2_b = 0, total = 0;
  int out_dim = 0, flat = 0;
};

ParamLayout param_layout(const ilsim_cnn_config& c);
void validate_config(const ilsim_cnn_config& c);
uint64_t param_count_of(const ilsim_cnn_config& c);
uint64_t model_flops_of(const ilsim_cnn_config& c);
int output_dim_of(const ilsim_cnn_config& c);
void init_weights_into(const ilsim_cnn_config& c, uint64_t seed, float* params);

// Floats per gathered sample row on the device: the 50*(mc+1) model input
// rounded up to whole conv0 windows (2 columns = 100 floats per row).
inline uint32_t input_row_floats(int max_context) {
  return 100u * static_cast<uint32_t>((max_context + 2) / 2);
}
// Device row layout of the gathered input per precision: bf16 rows are padded
// to 104 elements (208 B) so TMA row strides stay 16-B multiples.
inline uint32_t input_row_elems(int precision) { return precision == ILSIM_PREC_BF16 ? 104u : 100u; }
inline uint32_t input_stride(int max_context, int precision) {
  return input_row_elems(precision) * static_cast<uint32_t>((max_context + 2) / 2);
}
inline uint32_t input_elem_bytes(int precision) { return precision == ILSIM_PREC_BF16 ? 2u : 4u; }

struct TcModel;  // tensor-core operand copies (gemm_tc.cu)

struct DevModel {
  ilsim_cnn_config cfg{};
  ParamLayout L;
  DevBuf params;          // reference layout, f32
  TcModel* tc = nullptr;  // owned; null for the FP32 SIMT path
  DevModel() = default;
  DevModel(const DevModel&) = delete;
  DevModel& operator=(const DevModel&) = delete;
  ~DevModel();
};

struct ForwardBuffers {
  float* act[9];       // conv outputs (act[0..n_conv-1]), hidden (act[n_conv])
  float* y;            // head outputs
  uint32_t y_stride;
  uint32_t act_esz;    // bytes per conv activation element (2: bf16 tensor-core path)
  uint64_t part_off;   // first sample of this slice in the split-K partial buffer
  float* splitk;       // fp32 SIMT small-batch split-K scratch (null: tiled kernel only)
};

void model_upload(DevModel& m, const ilsim_cnn_config& c, const float* params, int precision,
                  cudaStream_t s);
ForwardBuffers forward_buffers(const DevModel& m, uint64_t chunk, DevBuf& act, DevBuf& y);
// The buffers of samples [off, ...) of a chunk: concurrent sub-trace groups
// each work on their own slice.
ForwardBuffers fb_slice(const DevModel& m, const ForwardBuffers& fb, uint64_t off);
// Runs the forward for `samples` gathered rows; returns kernels launched.
// With `fuse`, the tensor-core path also performs K3 (decode + clock) in its
// tail and returns true in *fused.
uint64_t forward_launch(const DevModel& m, int precision, const void* x, uint32_t x_stride,
                        uint64_t samples, const ForwardBuffers& fb, cudaStream_t s,
                        const DecodeParams* fuse = nullptr, bool* fused = nullptr, uint64_t x_lo_off = 0);
// True when the model's inference wants the gathered input pre-split into
// 3xTF32 hi / lo planes (tensor-core 3xTF32 with the fused conv chain).
bool split_input(const DevModel& m);

// tensor-core path (gemm_tc.cu)
TcModel* tc_model_create(const DevModel& m, const float* host_params, int precision, cudaStream_t s);
void tc_model_destroy(TcModel* t);
void tc_prepare(const DevModel& m, uint64_t samples);
uint64_t tc_forward(const DevModel& m, int precision, const void* x, uint32_t x_stride,
                    uint64_t samples, const ForwardBuffers& fb, cudaStream_t s, const DecodeParams* fuse,
                    uint64_t x_lo_off);
bool tc_split_input(const TcModel* t);
uint32_t tc_act_bytes(const TcModel* t);
// Fused round front available (C3 chain on the tensor-core path).
bool tc_fused_front(const TcModel* t);
void tc_calibrate(const DevModel& m, cudaStream_t s);
// K1 apply + gather + conv chain in one kernel (round_front.cu); the K1
// fields of fp are the caller's, the conv fields are filled in here.
uint64_t tc_front(const DevModel& m, FrontParams fp, const ForwardBuffers& fb, cudaStream_t s);
// FC1 + FC tail (+ fused K3 when fuse != null) on the flat conv output.
uint64_t tc_fc(const DevModel& m, const void* flat, uint64_t samples, const ForwardBuffers& fb, cudaStream_t s,
               const DecodeParams* fuse, bool with_tail);
// Where the fused round front finds the FC1 partials of a chunk (+ FC2 weights).
FcDecodeArgs tc_fc_decode_args(const DevModel& m, uint64_t samples, const ForwardBuffers& fb);

}  // namespace simnet
