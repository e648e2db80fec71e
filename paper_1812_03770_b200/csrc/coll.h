// Fused AllReduce + elementwise update over peer memory.
//
// The data-parallel step of the paper's graphs ends with ALLREDUCE_SUM of each
// gradient followed by the optimiser's elementwise update (W - lr * g) and an
// update edge ("natural support for parallel and distributed computing";
// P:283 update_iopair).  Here the sum over ranks and the update are ONE kernel:
// every rank maps the other ranks' graph pools (CUDA IPC over NVLink / NVSwitch),
// reads the gradient at the same pool offset on every rank (all ranks plan the same
// graph, so offsets agree), adds them in rank order 0..P-1 (deterministic and
// identical on every rank), applies the update's elementwise chain in registers
// and writes the updated value -- no separate NCCL call, no gradient round trip
// through HBM, no update kernel.  A cross-rank flag barrier (system-scope
// release/acquire on mapped flag words) orders the reads after every rank's
// gradient is final and keeps each rank's gradient alive until all peers have
// read it.  At world size 1 the kernel is the update alone (sum of one term).
#pragma once

#include <cuda_runtime.h>

#include "dot_tc.h"  // EpiProg (the elementwise chain interpreter's program)

namespace cg {

constexpr int kCollMaxRanks = 8;
constexpr int kCollFlagWords = 256;  // per rank: [0,64) arrive, [64,128) done, 128 epoch, 129 done counter

// one gradient: out[i] = chain( sum_{r = 0..P-1} g_r[i] ),  g_r = base[r] + goff
struct CollSeg {
  long long goff;   // gradient offset in floats from the pool base (equal on every rank)
  long long n;      // elements
  long long ncol;   // innermost extent (column operands of the chain)
  float* out;       // local result (the chain's sink, or the ALLREDUCE value itself)
  int vec;          // 16-byte vector path (n % 4 == 0, aligned)
  EpiProg epi;      // scalar: 0 column vector, 1 scalar, 2 full tensor
};

struct CollArgs {
  int nranks, rank;
  const float* base[kCollMaxRanks];           // every rank's pool base, mapped in this process
  unsigned long long* flags[kCollMaxRanks];   // every rank's flag words, mapped in this process
  const CollSeg* segs;                        // device table
  int nseg;
};

// One launch for a bucket of gradients (blockIdx.y = segment): one arrival barrier,
// the sums + chains, one departure barrier.
cudaError_t launch_fused_allreduce(const CollArgs& a, int num_sms, cudaStream_t s);
bool coll_seg_vec_ok(const CollSeg& s, const float* const* base, int nranks);

}  // namespace cg
