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
#include <cstdlib>
#include <cstdint>

#include "dot_small.h"
#include "kernels.h"

namespace cg {

namespace {

constexpr int NMAX = 32;

// ---- small N, ta = 0: A [M, K] row-major.  bs is op(B)^T with a padded row
// pitch (kc + 4: conflict-free staging stores, 16-byte aligned LDS.128); each
// warp keeps two rows in flight (row m and m + warps) so enough A bytes are
// outstanding per SM to cover HBM latency.
constexpr int RK = 8;  // float4 per lane per row held in registers (K <= 1024)
template <int NT>
__global__ void __launch_bounds__(NT >= 32 ? 256 : 512) dot_smalln_rows(const float* __restrict__ A, const float* __restrict__ B,
                                                       float* __restrict__ C, int M, int N, int K, int tb, int kc) {
  extern __shared__ float bs[];  // [NT][kc + 4] : op(B)^T chunk
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int warps = blockDim.x / 32;
  const int pitch = kc + 4;
  const bool vec = (K % 4) == 0;
  const bool one_chunk = K <= kc;
  auto stage = [&](int k0, int kn) {  // 8 loads in flight per thread (L2-latency bound otherwise)
    constexpr int U = 8;
    const int total = NT * kc;
    for (int e0 = threadIdx.x; e0 < total; e0 += U * blockDim.x) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * blockDim.x;
        int j, k;
        if (tb) j = e / kc, k = e % kc;  // B [N, K]: k contiguous
        else k = e / NT, j = e % NT;     // B [K, N]: j contiguous
        v[u] = (e < total && j < N && k < kn) ? __ldg(tb ? B + (size_t)j * K + k0 + k : B + (size_t)(k0 + k) * N + j) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * blockDim.x;
        int j, k;
        if (tb) j = e / kc, k = e % kc;
        else k = e / NT, j = e % NT;
        if (e < total) bs[j * pitch + k] = v[u];
      }
    }
  };
  const int mstride = gridDim.x * warps * 2;
  if (vec && K <= 128 * RK) {
    // Whole rows in registers: the first pair's loads are issued before op(B)
    // is staged (the HBM and L2 latencies overlap), the next pair's before the
    // shuffle reduction of the current one.
    float4 a[2][RK];
    auto load_rows = [&](int m0) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int m = m0 + r * warps + warp;
#pragma unroll
        for (int i = 0; i < RK; ++i) {
          const int k = lane * 4 + 128 * i;
          a[r][i] = (m < M && k < K) ? __ldg(reinterpret_cast<const float4*>(A + (size_t)m * K + k))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    };
    int m0 = blockIdx.x * warps * 2;
    if (m0 < M) load_rows(m0);
    stage(0, K);
    __syncthreads();
    for (; m0 < M; m0 += mstride) {
      float acc[2][NT];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[r][j] = 0.f;
#pragma unroll
      for (int i = 0; i < RK; ++i) {
        const int k = lane * 4 + 128 * i;
        if (k < K) {
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const float4 b = *reinterpret_cast<const float4*>(bs + j * pitch + k);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              acc[r][j] = fmaf(a[r][i].x, b.x, acc[r][j]);
              acc[r][j] = fmaf(a[r][i].y, b.y, acc[r][j]);
              acc[r][j] = fmaf(a[r][i].z, b.z, acc[r][j]);
              acc[r][j] = fmaf(a[r][i].w, b.w, acc[r][j]);
            }
          }
        }
      }
      if (m0 + mstride < M) load_rows(m0 + mstride);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int m = m0 + r * warps + warp;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          float v = acc[r][j];
#pragma unroll
          for (int o = 16; o >= 1; o /= 2) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
          acc[r][j] = v;
        }
        if (m < M && lane < NT && lane < N) {
          float v = 0.f;
#pragma unroll
          for (int j = 0; j < NT; ++j)
            if (j == lane) v = acc[r][j];
          C[(size_t)m * N + lane] = v;
        }
      }
    }
    return;
  }
  if (one_chunk) {
    stage(0, K);
    __syncthreads();
  }
  for (int m0 = blockIdx.x * warps * 2; m0 < M; m0 += mstride) {
    const int mr[2] = {m0 + warp, m0 + warps + warp};
    float acc[2][NT];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[r][j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += kc) {
      const int kn = min(kc, K - k0);
      if (!one_chunk) {
        __syncthreads();
        stage(k0, kn);
        __syncthreads();
      }
      if (vec) {
#pragma unroll 2
        for (int k = lane * 4; k < kn; k += 128) {
          float4 a[2];
#pragma unroll
          for (int r = 0; r < 2; ++r)
            a[r] = mr[r] < M ? __ldg(reinterpret_cast<const float4*>(A + (size_t)mr[r] * K + k0 + k))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const float4 b = *reinterpret_cast<const float4*>(bs + j * pitch + k);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              acc[r][j] = fmaf(a[r].x, b.x, acc[r][j]);
              acc[r][j] = fmaf(a[r].y, b.y, acc[r][j]);
              acc[r][j] = fmaf(a[r].z, b.z, acc[r][j]);
              acc[r][j] = fmaf(a[r].w, b.w, acc[r][j]);
            }
          }
        }
      } else {
        for (int k = lane; k < kn; k += 32) {
          float a[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) a[r] = mr[r] < M ? __ldg(A + (size_t)mr[r] * K + k0 + k) : 0.f;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const float b = bs[j * pitch + k];
#pragma unroll
            for (int r = 0; r < 2; ++r) acc[r][j] = fmaf(a[r], b, acc[r][j]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        float v = acc[r][j];
#pragma unroll
        for (int o = 16; o >= 1; o /= 2) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
        acc[r][j] = v;
      }
      if (mr[r] < M && lane < NT && lane < N) {
        float v = 0.f;
#pragma unroll
        for (int j = 0; j < NT; ++j)
          if (j == lane) v = acc[r][j];
        C[(size_t)mr[r] * N + lane] = v;
      }
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

// ---- small N, ta = 1, M % 4 == 0: each thread owns 4 consecutive m (one
// 128-bit load per k) and keeps 16 k-rows of A in flight; the block's whole
// k-chunk of op(B) is staged once.  Same per-(m, j) summation order as
// dot_smalln_cols (sequential k within the chunk, partials over chunks).
constexpr int C4_THREADS = 64, C4_U = 16, C4_KMAX = 256;
template <int NT>
__global__ void __launch_bounds__(C4_THREADS) dot_smalln_cols4(const float* __restrict__ A, const float* __restrict__ B,
                                                               float* __restrict__ out, int M, int N, int K, int tb,
                                                               int kchunk) {
  __shared__ __align__(16) float bs[C4_KMAX][NT];
  const int m = (blockIdx.x * C4_THREADS + threadIdx.x) * 4;
  const int kb = blockIdx.y * kchunk, kn = min(K, kb + kchunk) - kb;
  for (int e0 = threadIdx.x; e0 < kchunk * NT; e0 += 8 * C4_THREADS) {  // 8 L2 loads in flight per thread
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * C4_THREADS, k = e / NT, j = e % NT;
      v[u] = (e < kchunk * NT && j < N && k < kn) ? __ldg(tb ? B + (size_t)j * K + kb + k : B + (size_t)(kb + k) * N + j)
                                                  : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * C4_THREADS;
      if (e < kchunk * NT) bs[e / NT][e % NT] = v[u];
    }
  }
  __syncthreads();
  if (m >= M) return;
  float acc[4][NT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j] = 0.f;
  const float* a0 = A + (size_t)kb * M + m;
  int k = 0;
  for (; k + C4_U <= kn; k += C4_U) {
    float4 a[C4_U];
#pragma unroll
    for (int q = 0; q < C4_U; ++q) a[q] = __ldg(reinterpret_cast<const float4*>(a0 + (size_t)(k + q) * M));
#pragma unroll
    for (int q = 0; q < C4_U; ++q)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const float b = bs[k + q][j];
        acc[0][j] = fmaf(a[q].x, b, acc[0][j]);
        acc[1][j] = fmaf(a[q].y, b, acc[1][j]);
        acc[2][j] = fmaf(a[q].z, b, acc[2][j]);
        acc[3][j] = fmaf(a[q].w, b, acc[3][j]);
      }
  }
  for (; k < kn; ++k) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(a0 + (size_t)k * M));
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const float b = bs[k][j];
      acc[0][j] = fmaf(a.x, b, acc[0][j]);
      acc[1][j] = fmaf(a.y, b, acc[1][j]);
      acc[2][j] = fmaf(a.z, b, acc[2][j]);
      acc[3][j] = fmaf(a.w, b, acc[3][j]);
    }
  }
  float* o = out + (size_t)blockIdx.y * M * N + (size_t)m * N;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
      if (j < N) o[i * N + j] = acc[i][j];
}

// ---- small K: C[m, n..n+3] = sum_k A(m,k) B(k, n..n+3); block = 64 n-quads x 4 rows
constexpr int SK_TN = 256;  // columns per block
template <int KT>  // KT > 0: the inner extent at compile time (no predicated 32-long loops)
__global__ void __launch_bounds__(256) dot_smallk(const float* __restrict__ A, const float* __restrict__ B,
                                                  float* __restrict__ C, int M, int N, int K_, int ta, int tb) {
  constexpr int KMAX = KT > 0 ? KT : 32;
  const int K = KT > 0 ? KT : K_;
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
    float a[RPT][KMAX];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int m = mb + i;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        a[i][k] = (k < K && m < M) ? __ldg(ta ? A + (size_t)k * M + m : A + (size_t)m * K + k) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int m = mb + i;
      if (m >= M) break;
      float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
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
  const size_t smem = (size_t)NT * (kc + 4) * sizeof(float);
  const cudaError_t ae = smem_attr((const void*)dot_smalln_rows<NT>, 227 * 1024);  // per device
  if (ae != cudaSuccess) return ae;
  // one 16-warp block per SM: op(B)^T is staged once per SM (not once per 16 rows --
  // the staging was the kernel's cost) and every warp walks its rows two at a time
  const int warps = NT >= 32 ? 8 : 16;  // (32 accumulators x 2 rows need the registers of 8 warps)
  const int blocks_per_sm = warps >= 16 ? 1 : std::max(1, std::min(4, (int)(227 * 1024 / std::max<size_t>(smem, 1))));
  int grid = std::min((M + 2 * warps - 1) / (2 * warps), num_sms * blocks_per_sm);
  dot_smalln_rows<NT><<<grid, warps * 32, smem, s>>>(A, B, C, M, N, K, tb, kc);
  return cudaGetLastError();
}

bool cols4_ok(const float* A, int M) { return M % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0; }

void cols4_split(int M, int K, int num_sms, int* kchunk, int* S) {
  const int mblocks = (M + 4 * C4_THREADS - 1) / (4 * C4_THREADS);
  // ~8 blocks (16 warps) per SM, k-chunks of >= 32 rows (partials stay << the A read)
  int s = std::max(1, std::min((8 * num_sms + mblocks - 1) / mblocks, (K + 31) / 32));
  int ch = (K + s - 1) / s;
  ch = std::min(C4_KMAX, (ch + C4_U - 1) / C4_U * C4_U);
  *kchunk = ch;
  *S = (K + ch - 1) / ch;
}

template <int NT>
cudaError_t launch_cols(const float* A, const float* B, float* C, float* ws, int M, int N, int K, int tb, int num_sms,
                        cudaStream_t s) {
  int kchunk, S;
  if (cols4_ok(A, M)) {
    cols4_split(M, K, num_sms, &kchunk, &S);
    dim3 grid((M + 4 * C4_THREADS - 1) / (4 * C4_THREADS), S);
    dot_smalln_cols4<NT><<<grid, C4_THREADS, 0, s>>>(A, B, S > 1 ? ws : C, M, N, K, tb, kchunk);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || S == 1) return e;
    return launch_reduce_finalize(ws, C, (long long)M * N, S, 0, s);
  }
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
  int kchunk, S, kchunk4, S4;
  cols_split(M, K, num_sms, &kchunk, &S);
  cols4_split(M, K, num_sms, &kchunk4, &S4);  // either variant may run (alignment is known at launch)
  S = std::max(S, S4);
  return S > 1 ? (size_t)S * M * N : 0;
}

cudaError_t launch_dot_small(const float* A, const float* B, float* C, float* ws, int M, int N, int K, int ta, int tb,
                             int num_sms, cudaStream_t s) {
  const int kind = dot_small_kind(M, N, K);
  if (kind == DOT_SMALL_K) {
    const int gx = (N + SK_TN - 1) / SK_TN;
    dim3 grid(gx, std::min((M + 3) / 4, std::max(1, num_sms * 6 / gx)));  // one full wave (32 KB smem / block)
    if (K == 10) dot_smallk<10><<<grid, 256, 0, s>>>(A, B, C, M, N, K, ta, tb);  // logits width of C3 / C4
    else if (K <= 16) dot_smallk<16><<<grid, 256, 0, s>>>(A, B, C, M, N, K, ta, tb);
    else dot_smallk<0><<<grid, 256, 0, s>>>(A, B, C, M, N, K, ta, tb);
    return cudaGetLastError();
  }
  if (kind != DOT_SMALL_N) return cudaErrorInvalidValue;
  if (!ta) {
    if (N <= 8) return launch_rows<8>(A, B, C, M, N, K, tb, num_sms, s);
    if (N <= 12) return launch_rows<12>(A, B, C, M, N, K, tb, num_sms, s);
    if (N <= 16) return launch_rows<16>(A, B, C, M, N, K, tb, num_sms, s);
    return launch_rows<32>(A, B, C, M, N, K, tb, num_sms, s);
  }
  if (N <= 8) return launch_cols<8>(A, B, C, ws, M, N, K, tb, num_sms, s);
  if (N <= 12) return launch_cols<12>(A, B, C, ws, M, N, K, tb, num_sms, s);
  if (N <= 16) return launch_cols<16>(A, B, C, ws, M, N, K, tb, num_sms, s);
  return launch_cols<32>(A, B, C, ws, M, N, K, tb, num_sms, s);
}

}  // namespace cg
