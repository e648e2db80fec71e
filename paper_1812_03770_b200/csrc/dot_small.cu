// DOT nodes with one small extent (HBM-bound products: logits, their gradients,
// rank-10 updates).  C[M,N] = op(A)[M,K] . op(B)[K,N], fp32 FFMA accumulation in
// a fixed order (deterministic, no atomics).  These shapes have arithmetic
// intensity of at most ~N/2 FLOP/B, so the design goal is one pass over the
// large operand at HBM speed, not tensor-core throughput:
//
//   small N (N <= 32), A K-contiguous (ta = 0): one warp per row of A; the
//       row streams through 128-bit loads, op(B) sits transposed in shared
//       memory (BsT[j][k]) so each lane reads its 4 k-values of column j with
//       one conflict-free LDS.128; N partial sums per lane, fixed-order shuffle tree.
//   small N, A M-contiguous (ta = 1): threads over m (coalesced), sequential k
//       with op(B)[k][0..N) broadcast from shared memory; K is split over
//       grid.y into workspace partials reduced by a fixed-order finalize.
//   small K (K <= 32): output-bound; op(B) tile staged in shared memory, each
//       thread writes 4 consecutive outputs of one row (128-bit store).
#include <cuda_runtime.h>

#include <algorithm>

#include "dot_small.h"
#include "kernels.h"

namespace cg {

namespace {

constexpr int NMAX = 32;

// ---- small N, ta = 0: A [M, K] row-major
template <int NT>
__global__ void __launch_bounds__(256) dot_smalln_rows(const float* __restrict__ A, const float* __restrict__ B,
                                                       float* __restrict__ C, int M, int N, int K, int tb, int kc) {
  extern __shared__ float bs[];  // [NT][kc] : op(B)^T chunk
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int warps = blockDim.x / 32;
  const bool vec = (K % 4) == 0;
  const bool one_chunk = K <= kc;
  auto stage = [&](int k0, int kn) {
    for (int e = threadIdx.x; e < NT * kc; e += blockDim.x) {
      const int j = e / kc, k = e % kc;
      float v = 0.f;
      if (j < N && k < kn) v = tb ? B[(size_t)j * K + k0 + k] : B[(size_t)(k0 + k) * N + j];
      bs[e] = v;
    }
  };
  if (one_chunk) {
    stage(0, K);
    __syncthreads();
  }
  for (int m0 = blockIdx.x * warps; m0 < M; m0 += gridDim.x * warps) {
    const int m = m0 + warp;
    float acc[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += kc) {
      const int kn = min(kc, K - k0);
      if (!one_chunk) {
        __syncthreads();
        stage(k0, kn);
        __syncthreads();
      }
      if (m < M) {
        const float* arow = A + (size_t)m * K + k0;
        if (vec) {
          for (int k = lane * 4; k < kn; k += 128) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(arow + k));
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              const float4 b = *reinterpret_cast<const float4*>(bs + j * kc + k);
              acc[j] = fmaf(a.x, b.x, acc[j]);
              acc[j] = fmaf(a.y, b.y, acc[j]);
              acc[j] = fmaf(a.z, b.z, acc[j]);
              acc[j] = fmaf(a.w, b.w, acc[j]);
            }
          }
        } else {
          for (int k = lane; k < kn; k += 32) {
            const float a = __ldg(arow + k);
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[j] = fmaf(a, bs[j * kc + k], acc[j]);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      float v = acc[j];
#pragma unroll
      for (int o = 16; o >= 1; o /= 2) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
      acc[j] = v;
    }
    if (m < M && lane < NT && lane < N) {
      float v = 0.f;
#pragma unroll
      for (int j = 0; j < NT; ++j)
        if (j == lane) v = acc[j];
      C[(size_t)m * N + lane] = v;
    }
  }
}

// ---- small N, ta = 1: A stored [K, M] (M contiguous); partials over K chunks
template <int NT>
__global__ void __launch_bounds__(256) dot_smalln_cols(const float* __restrict__ A, const float* __restrict__ B,
                                                       float* __restrict__ out, int M, int N, int K, int tb, int kchunk) {
  __shared__ float bs[64][NT];
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int kb = blockIdx.y * kchunk, ke = min(K, kb + kchunk);
  float acc[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j] = 0.f;
  for (int k0 = kb; k0 < ke; k0 += 64) {
    const int kn = min(64, ke - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * NT; e += blockDim.x) {
      const int k = e / NT, j = e % NT;
      float v = 0.f;
      if (j < N && k < kn) v = tb ? B[(size_t)j * K + k0 + k] : B[(size_t)(k0 + k) * N + j];
      bs[k][j] = v;
    }
    __syncthreads();
    if (m < M) {
      int k = 0;
      for (; k + 8 <= kn; k += 8) {  // 8 independent loads in flight, then the FMAs in k order
        float a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = __ldg(A + (size_t)(k0 + k + q) * M + m);
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[j] = fmaf(a[q], bs[k + q][j], acc[j]);
      }
      for (; k < kn; ++k) {
        const float a = __ldg(A + (size_t)(k0 + k) * M + m);
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[j] = fmaf(a, bs[k][j], acc[j]);
      }
    }
  }
  if (m < M) {
    float* o = out + (size_t)blockIdx.y * M * N + (size_t)m * N;
#pragma unroll
    for (int j = 0; j < NT; ++j)
      if (j < N) o[j] = acc[j];
  }
}

// ---- small K: C[m, n..n+3] = sum_k A(m,k) B(k, n..n+3); block = 64 n-quads x 4 rows
constexpr int SK_TN = 256;  // columns per block
__global__ void __launch_bounds__(256) dot_smallk(const float* __restrict__ A, const float* __restrict__ B,
                                                  float* __restrict__ C, int M, int N, int K, int ta, int tb) {
  __shared__ float bs[32][SK_TN];
  const int n0 = blockIdx.x * SK_TN;
  for (int e = threadIdx.x; e < K * SK_TN; e += blockDim.x) {
    const int k = e / SK_TN, n = e % SK_TN;
    float v = 0.f;
    if (n0 + n < N) v = tb ? B[(size_t)(n0 + n) * K + k] : B[(size_t)k * N + n0 + n];
    bs[k][n] = v;
  }
  __syncthreads();
  const int q = threadIdx.x % 64, r = threadIdx.x / 64;
  const int n = n0 + q * 4;
  const bool vec = (N % 4) == 0;
  // RPT rows per thread per iteration: all A loads of those rows first (ILP)
  constexpr int RPT = 1;
  for (int mb = (blockIdx.y * 4 + r) * RPT; mb < M; mb += gridDim.y * 4 * RPT) {
    float a[RPT][32];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int m = mb + i;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        a[i][k] = (k < K && m < M) ? __ldg(ta ? A + (size_t)k * M + m : A + (size_t)m * K + k) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int m = mb + i;
      if (m >= M) break;
      float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < K) {
          const float4 b = *reinterpret_cast<const float4*>(&bs[k][q * 4]);
          c0 = fmaf(a[i][k], b.x, c0);
          c1 = fmaf(a[i][k], b.y, c1);
          c2 = fmaf(a[i][k], b.z, c2);
          c3 = fmaf(a[i][k], b.w, c3);
        }
      }
      float* crow = C + (size_t)m * N;
      if (vec && n + 4 <= N) {
        *reinterpret_cast<float4*>(crow + n) = make_float4(c0, c1, c2, c3);
      } else {
        if (n < N) crow[n] = c0;
        if (n + 1 < N) crow[n + 1] = c1;
        if (n + 2 < N) crow[n + 2] = c2;
        if (n + 3 < N) crow[n + 3] = c3;
      }
    }
  }
}

// k-chunk of op(B)^T kept in shared memory: at most 192 KiB
int rows_kchunk(int K, int nt) { return std::min(((K + 127) / 128) * 128, (49152 / nt) / 128 * 128); }

void cols_split(int M, int K, int num_sms, int* kchunk, int* S) {
  const int mblocks = (M + 255) / 256;
  int s = std::max(1, std::min((2 * num_sms + mblocks - 1) / mblocks, (K + 63) / 64));
  int ch = (K + s - 1) / s;
  ch = (ch + 63) / 64 * 64;
  *kchunk = ch;
  *S = (K + ch - 1) / ch;
}

template <int NT>
cudaError_t launch_rows(const float* A, const float* B, float* C, int M, int N, int K, int tb, int num_sms, cudaStream_t s) {
  const int kc = rows_kchunk(K, NT);
  const size_t smem = (size_t)NT * kc * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dot_smalln_rows<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int warps = 8;
  // few blocks, many rows each: op(B)^T is staged once per block and reused
  const int blocks_per_sm = std::max(1, std::min(4, (int)(227 * 1024 / std::max<size_t>(smem, 1))));
  int grid = std::min((M + warps - 1) / warps, num_sms * blocks_per_sm);
  dot_smalln_rows<NT><<<grid, warps * 32, smem, s>>>(A, B, C, M, N, K, tb, kc);
  return cudaGetLastError();
}

template <int NT>
cudaError_t launch_cols(const float* A, const float* B, float* C, float* ws, int M, int N, int K, int tb, int num_sms,
                        cudaStream_t s) {
  int kchunk, S;
  cols_split(M, K, num_sms, &kchunk, &S);
  dim3 grid((M + 255) / 256, S);
  dot_smalln_cols<NT><<<grid, 256, 0, s>>>(A, B, S > 1 ? ws : C, M, N, K, tb, kchunk);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || S == 1) return e;
  return launch_reduce_finalize(ws, C, (long long)M * N, S, 0, s);
}

}  // namespace

int dot_small_kind(int M, int N, int K) {
  if (N <= NMAX) return DOT_SMALL_N;
  if (K <= 32) return DOT_SMALL_K;
  return DOT_SMALL_NONE;
}

size_t dot_small_ws_floats(int M, int N, int K, int ta, int num_sms) {
  if (dot_small_kind(M, N, K) != DOT_SMALL_N || !ta) return 0;
  int kchunk, S;
  cols_split(M, K, num_sms, &kchunk, &S);
  return S > 1 ? (size_t)S * M * N : 0;
}

cudaError_t launch_dot_small(const float* A, const float* B, float* C, float* ws, int M, int N, int K, int ta, int tb,
                             int num_sms, cudaStream_t s) {
  const int kind = dot_small_kind(M, N, K);
  if (kind == DOT_SMALL_K) {
    const int gx = (N + SK_TN - 1) / SK_TN;
    dim3 grid(gx, std::min((M + 3) / 4, std::max(1, num_sms * 6 / gx)));  // one full wave (32 KB smem / block)
    dot_smallk<<<grid, 256, 0, s>>>(A, B, C, M, N, K, ta, tb);
    return cudaGetLastError();
  }
  if (kind != DOT_SMALL_N) return cudaErrorInvalidValue;
  if (!ta) {
    if (N <= 8) return launch_rows<8>(A, B, C, M, N, K, tb, num_sms, s);
    if (N <= 16) return launch_rows<16>(A, B, C, M, N, K, tb, num_sms, s);
    return launch_rows<32>(A, B, C, M, N, K, tb, num_sms, s);
  }
  if (N <= 8) return launch_cols<8>(A, B, C, ws, M, N, K, tb, num_sms, s);
  if (N <= 16) return launch_cols<16>(A, B, C, ws, M, N, K, tb, num_sms, s);
  return launch_cols<32>(A, B, C, ws, M, N, K, tb, num_sms, s);
}

}  // namespace cg
