// DOT nodes with one small extent (dot_small.cu): SIMT, HBM-bound, deterministic.
#pragma once

#include <cstddef>

#include <cuda_runtime.h>

namespace cg {

enum { DOT_SMALL_NONE = 0, DOT_SMALL_N = 1, DOT_SMALL_K = 2 };

// Which small-extent kernel serves C[M,N] = op(A) op(B) with inner extent K
// (N <= 32: small N; else K <= 32: small K; else none).
int dot_small_kind(int M, int N, int K);
// Workspace (floats) for the split-K partials of the small-N, ta = 1 kernel.
size_t dot_small_ws_floats(int M, int N, int K, int ta, int num_sms);
cudaError_t launch_dot_small(const float* A, const float* B, float* C, float* ws, int M, int N, int K, int ta, int tb,
                             int num_sms, cudaStream_t s);

}  // namespace cg
