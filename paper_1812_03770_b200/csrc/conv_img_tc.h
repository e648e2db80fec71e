// Few-channel, small-image convolutions on the tensor cores (conv_img_tc.cu):
// the forward correlation and the backward-input pass (as a correlation of dy
// with the flipped, transposed kernel) of C4's LeNet shapes.
#pragma once

#include <cuda_runtime.h>

#include "kernels.h"

namespace cg {

struct EpiProg;

// true when (geometry, pass) has a compiled instantiation; flip = backward-input
bool conv_img_tc_supported(const ConvGeom& g, bool flip);
// fwd:  y[n,oh,ow,co] = sum_{kh,kw,ci} x[n,oh+kh-pt,ow+kw-pl,ci] w[kh,kw,ci,co]
// flip: dx[n,h,w,ci]  = sum_{kh,kw,co} dy[n,h-kh+pt,w-kw+pl,co] w[kh,kw,ci,co]   (stride 1)
// epi (forward only; NULL or n == 0: plain store): the fused elementwise chain of
// the f2 epilogue fusion, applied to each output pixel's COUT values before the store
cudaError_t launch_conv_img_tc(const float* in, const float* w, float* out, const ConvGeom& g, bool flip, int num_sms,
                               cudaStream_t s, const EpiProg* epi = nullptr);

// backward-kernel (C4 geometries; g = the forward conv): dw[kh,kw,ci,co] =
// sum_{n,oh,ow} x[n,oh+kh-pt,ow+kw-pl,ci] dy[n,oh,ow,co]; per-CTA partials in ws
// (conv_img_tc_bwdk_ws floats), summed in a fixed order into dw
// db != NULL (conv_img_tc_bwdk_bias_ok): also db[co] = sum_{n,oh,ow} dy[n,oh,ow,co] from
// the same dy reads (a SUM group fused into this one)
bool conv_img_tc_bwdk_supported(const ConvGeom& g);
bool conv_img_tc_bwdk_bias_ok(const ConvGeom& g);
size_t conv_img_tc_bwdk_ws(const ConvGeom& g, int num_sms);
// pcodes != NULL (same geometries): dy = RELU_GRAD(a, MAXPOOL2D_BWD(relu(a), dp)) given
// as dp (pointer `dy`, [n, ho/2, wo/2, co]) and the pool's decision codes (launch_maxpool)
cudaError_t launch_conv_img_tc_bwdk(const float* x, const float* dy, float* dw, float* ws, const ConvGeom& g, int num_sms,
                                    cudaStream_t s, float* db = nullptr, const unsigned char* pcodes = nullptr);

// The InceptionV3 stem conv (Ci = 3, stride 2) over bands of output rows, with the
// DOT/CONV epilogue's fused elementwise chain (conv_band_tc_kernel); x must be
// 16-byte aligned and may be over-read by up to 12 bytes inside its allocation.
bool conv_band_supported(int n, int h, int w, int ci, int kh, int kw, int co, int ho, int wo, int sh, int sw, int pt,
                         int pl);
cudaError_t launch_conv_band(const float* x, const float* w, float* out, int ldc, int n, const EpiProg& epi, int num_sms,
                             cudaStream_t s);
// 3x3 stride-1 convs with 32 input channels on wide images (the InceptionV3 stem's
// layers 2 and 3): input rows staged once each in a ring (conv_rows_tc_kernel).
// kind 0 = not compiled for this geometry.
int conv_rows_kind(int h, int w, int ci, int kh, int kw, int co, int ho, int wo, int sh, int sw, int pt, int pl);
cudaError_t launch_conv_rows(int kind, const float* x, const float* w, float* out, int ldc, int n, const EpiProg& epi,
                             int num_sms, cudaStream_t s);

}  // namespace cg
