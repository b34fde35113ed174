// [EXT] CNN stages on the tcgen05 tensor cores (conv_tc.cu): implicit-GEMM forward, input-delta
// and weight-gradient (+ fused leapfrog) contractions over NHWC activation buffers.
#pragma once

#include "ctx.cuh"

namespace dasmc_b200 {

bool cnn_tc_eligible(const Ctx& c);
void cnn_tc_init(Ctx& c);
void cnn_tc_free(Ctx& c);
void cnn_tc_refresh_data(Ctx& c, const float* X, int64_t rows);  // tf32 copy of the stage-0 input rows
int64_t cnn_tc_image_floats(const Ctx& c);  // stage-buffer floats per (image, particle)
void cnn_tc_alloc(Ctx& c, int64_t mc);      // stage buffers + operand tables for chunks of mc images
float* cnn_tc_flat(Ctx& c);                 // [Jmax][mcap][F] head input / its delta
void cnn_tc_weights(Ctx& c, const float* theta, int64_t J, bool need_grad);
void cnn_tc_forward(Ctx& c, const float* theta, int64_t J, int64_t m0, int64_t mc);
void cnn_tc_backward(Ctx& c, const float* theta, int64_t J, int64_t m0, int64_t mc, const EpiParams& e);

}  // namespace dasmc_b200
