// Hand-written (precompiled, sm_100a) kernels used by the executor.
// Every launcher enqueues on the given stream and returns the launch status.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace cg {

struct CopyDesc {  // one update edge / copy: dst[0:n] <- src[0:n]
  const float* src;
  float* dst;
  long long n;
};

// Single-pass update-edge copy [update_iopair, P:283]: all descriptors in one launch.
cudaError_t launch_update_copy(const CopyDesc* descs_dev, int n_desc, long long max_n, cudaStream_t s);
// Row-major copy (RESHAPE that cannot slide in place; ALLREDUCE_SUM at world 1).
cudaError_t launch_copy(const float* src, float* dst, long long n, cudaStream_t s);
// Fixed-order reduction of S split partials: out[j] = op_{s<S} ws[s*OI + j]  (op: 0 sum, 1 max).
cudaError_t launch_reduce_finalize(const float* ws, float* out, long long oi, long long S, int op, cudaStream_t s);

// DOT: C[M,N] = op(A) op(B), fp32 in/out, fp32 FFMA accumulation (SIMT).
cudaError_t launch_dot_simt(const float* A, const float* B, float* C, int M, int N, int K, int ta, int tb,
                            cudaStream_t s);

// CONV2D family / pools / concat (NHWC activations, HWIO kernels)
struct ConvGeom {
  int n, h, w, ci, kh, kw, co, ho, wo, sh, sw, pt, pl;
};
cudaError_t launch_conv2d_fwd(const float* x, const float* w, float* y, const ConvGeom& g, cudaStream_t s);
cudaError_t launch_conv2d_bwd_input(const float* dy, const float* w, float* dx, const ConvGeom& g, cudaStream_t s);
// returns the workspace (floats) it needs when ws == nullptr
size_t conv2d_bwd_kernel_ws(const ConvGeom& g, int num_sms);
cudaError_t launch_conv2d_bwd_kernel(const float* x, const float* dy, float* dw, float* ws, const ConvGeom& g,
                                     int num_sms, cudaStream_t s);
struct EpiProg;
// f2 pooling fusion (2 x 2 stride-2 pools over few channels, even H and W):
// launch_maxpool with `pro` first computes its input from `x` by the fused
// elementwise chain of the producing group (xo = pro(x), written in full) and pools
// that; launch_maxpool_bwd with `epi` applies the consuming group's chain to every
// gradient value before the store.  NULL / n == 0: the plain kernels.
bool maxpool_fusable(const ConvGeom& g);
// codes (maxpool_fusable geometries): one byte per (output pixel, channel), the window
// position the backward pass routes the gradient to -- written by the forward
// kernel, read by the backward kernel instead of the input's four window values.
cudaError_t launch_maxpool(const float* x, float* y, const ConvGeom& g, cudaStream_t s, const EpiProg* pro = nullptr,
                           float* xo = nullptr, unsigned char* codes = nullptr);
// code_mask (with codes): the consumer RELU_GRAD(a, .) of a pool over relu(a), applied
// from the codes' recorded sign bit (a is not read)
cudaError_t launch_maxpool_bwd(const float* x, const float* dy, float* dx, const ConvGeom& g, cudaStream_t s,
                               const EpiProg* epi = nullptr, const unsigned char* codes = nullptr, int code_mask = 0);
cudaError_t launch_avgpool(const float* x, float* y, const ConvGeom& g, cudaStream_t s);

constexpr int kMaxConcat = 16;
struct ConcatArgs {
  const float* src[kMaxConcat];
  long long inner[kMaxConcat];   // elements per outer index contributed by each source
  long long offset[kMaxConcat];  // element offset of each source inside a destination row
  int n;                         // sources: they need not cover the row (R14 slices stay untouched)
};
cudaError_t launch_concat(const ConcatArgs& a, float* dst, long long outer, long long dst_inner, cudaStream_t s);

// cudaFuncAttributeMaxDynamicSharedMemorySize for kernel fn on the CURRENT device,
// set once per (kernel, device, bytes): the attribute is per device, so a process
// driving graphs on several devices must set it on each of them (thread-safe).
cudaError_t smem_attr(const void* fn, int bytes);

// Debug only (CG_DEBUG_CLOBBER): checksum of n floats, synchronous on stream s.
unsigned long long debug_checksum(const float* p, long long n, cudaStream_t s);

}  // namespace cg
