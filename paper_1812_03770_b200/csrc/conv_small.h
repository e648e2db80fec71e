// CONV2D family for small images / few channels with whole images in shared
// memory (conv_small.cu).  *_ok() say whether a geometry fits.
#pragma once

#include <cstddef>

#include <cuda_runtime.h>

#include "kernels.h"

namespace cg {

bool conv_small_fwd_ok(const ConvGeom& g);
bool conv_small_bwdin_ok(const ConvGeom& g);
bool conv_small_bwdk_ok(const ConvGeom& g);
size_t conv_small_bwdk_ws(const ConvGeom& g, int num_sms);  // floats of per-block partials
cudaError_t launch_conv_small_fwd(const float* x, const float* w, float* y, const ConvGeom& g, int num_sms, cudaStream_t s);
cudaError_t launch_conv_small_bwdin(const float* dy, const float* w, float* dx, const ConvGeom& g, int num_sms,
                                    cudaStream_t s);
cudaError_t launch_conv_small_bwdk(const float* x, const float* dy, float* dw, float* ws, const ConvGeom& g,
                                   int num_sms, cudaStream_t s);

}  // namespace cg
