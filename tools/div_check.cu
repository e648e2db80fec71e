// Bit-exactness check of div_rn_n (dot_tc.h) against __fdiv_rn on random operands.
#include <cstdio>
#include <cstdint>
#include "../paper_1812_03770_b200/csrc/dot_tc.h"
using namespace cg;
__device__ unsigned long long mismatches, checked_fast;
__global__ void k(unsigned long long seed, int mode) {
  unsigned long long s = seed ^ (blockIdx.x * 0x9E3779B97F4A7C15ull + threadIdx.x * 0xBF58476D1CE4E5B9ull);
  for (int it = 0; it < 256; ++it) {
    float a[16], b[16], v[16];
    for (int i = 0; i < 16; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      unsigned ua = (unsigned)s, ub = (unsigned)(s >> 32);
      if (mode == 0) {  // exponents near 1 (BN-like)
        ua = (ua & 0x807FFFFFu) | ((120u + (ua >> 27) % 16u) << 23);
        ub = (ub & 0x807FFFFFu) | ((120u + (ub >> 27) % 16u) << 23);
      } else if (mode == 1) {  // full exponent range near the limits
        ua = (ua & 0x807FFFFFu) | ((((ua >> 23) & 255u) % 210u + 22u) << 23);
        ub = (ub & 0x807FFFFFu) | ((((ub >> 23) & 255u) % 210u + 22u) << 23);
      } else if (mode == 3) {  // the fast path's whole exponent window [-60, 60]
        ua = (ua & 0x807FFFFFu) | ((((ua >> 23) & 255u) % 121u + 67u) << 23);
        ub = (ub & 0x807FFFFFu) | ((((ub >> 23) & 255u) % 121u + 67u) << 23);
      }  // mode 2: raw bits (inf, NaN, denormal, zero included)
      a[i] = __uint_as_float(ua); b[i] = __uint_as_float(ub); v[i] = a[i];
    }
    div_rn_n<16>(v, b, false);
    for (int i = 0; i < 16; ++i) {
      const float ref = __fdiv_rn(a[i], b[i]);
      const bool same = __float_as_uint(ref) == __float_as_uint(v[i]) || (ref != ref && v[i] != v[i]);
      if (!same) atomicAdd(&mismatches, 1ull);
    }
    atomicAdd(&checked_fast, 16ull);
  }
}
int main() {
  for (int mode = 0; mode < 4; ++mode) {
    unsigned long long z = 0, m = 0, c = 0;
    cudaMemcpyToSymbol(mismatches, &z, 8); cudaMemcpyToSymbol(checked_fast, &z, 8);
    for (int rep = 0; rep < 8; ++rep) k<<<1184, 256>>>(1234567ull + rep * 7919ull + mode, mode);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&m, mismatches, 8); cudaMemcpyFromSymbol(&c, checked_fast, 8);
    printf("mode %d: %llu divisions, %llu mismatches vs __fdiv_rn\n", mode, c, m);
  }
  return 0;
}
