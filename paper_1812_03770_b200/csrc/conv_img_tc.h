// Few-channel, small-image convolutions on the tensor cores (conv_img_tc.cu):
// the forward correlation and the backward-input pass (as a correlation of dy
// with the flipped, transposed kernel) of C4's LeNet shapes.
#pragma once

#include <cuda_runtime.h>

#include "kernels.h"

namespace cg {

// true when (geometry, pass) has a compiled instantiation; flip = backward-input
bool conv_img_tc_supported(const ConvGeom& g, bool flip);
// fwd:  y[n,oh,ow,co] = sum_{kh,kw,ci} x[n,oh+kh-pt,ow+kw-pl,ci] w[kh,kw,ci,co]
// flip: dx[n,h,w,ci]  = sum_{kh,kw,co} dy[n,h-kh+pt,w-kw+pl,co] w[kh,kw,ci,co]   (stride 1)
cudaError_t launch_conv_img_tc(const float* in, const float* w, float* out, const ConvGeom& g, bool flip, int num_sms,
                               cudaStream_t s);

}  // namespace cg
