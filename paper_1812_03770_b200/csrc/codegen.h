// Code generator: one CUDA C++ kernel per fused elementwise / reduction group,
// compiled with NVRTC for sm_100a (runtime.cu).  Pure host code.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "host.h"

namespace cg {

struct KernelSpec {
  std::string name;     // extern "C" symbol (hash of the body)
  std::string source;   // complete translation unit
  uint32_t grid[3] = {1, 1, 1};
  uint32_t block = 256;
  int64_t work_blocks = 1;   // grid-stride kernels: blocks that still have work (upper bound for grid.x)
  std::vector<int> in_ids;   // kernel args: input pointers (group inputs order)
  std::vector<int> out_ids;  // then output pointers (materialised values, gamma order)
  bool uses_ws = false;      // last arg: float* workspace (reduction partials)
  // reduction finalize (SUM/MAX over S partials of O*I values, fixed order)
  int64_t splits = 1, oi = 0;
  int red_op = 0;            // CG_SUM / CG_MAX
  int red_out = -1;          // node id of the reduction sink
  uint64_t ws_floats = 0;
  std::string mode;          // "row", "flat", "red" (for reports)
};

// Generate the kernel of an elementwise (G_EW) or reduction (G_RED) group.
KernelSpec gen_group(const HostGraph& hg, const Group& G, int num_sms);

// One kernel for a run of consecutive EW / row-reduction groups over a [B, N]
// domain (warp per row; f2 reduce -> broadcast fusion, e.g. softmax).  Empty name:
// the run does not qualify.
KernelSpec gen_rowrun(const HostGraph& hg, const std::vector<const Group*>& run, int num_sms);

}  // namespace cg
