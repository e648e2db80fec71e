// Executor order with batched collectives (data-parallel training).
//
// Gamma [P:312] interleaves each gradient's ALLREDUCE_SUM with the SGD group that
// consumes it ("AR(dW1) SGD(W1) SUM(db1) AR(db1) SGD(b1) DOT(dW2) ..."), so issuing
// the groups in Gamma order gives one latency-bound collective per gradient.
// collective_schedule() defers every collective, and every group that reads a
// deferred group's output, for as long as no later group touches a block they read
// or write; the deferred groups are then issued with all mutually independent
// collectives in ONE step (one ncclGroupStart/End, one fused NCCL launch).
//
// Validity: the result is a permutation of the active groups in which every pair
// of groups that conflict — one writes a pool block the other reads or writes
// (Alg. 1 reuses blocks, so write-after-read matters), or both use the kernel
// workspace — keeps its Gamma order, and groups sharing a step are collectives
// with no conflict between them.  Any such permutation computes the same values
// as Gamma order (conflict-free groups commute).
#pragma once

#include <vector>

namespace cg {

// rd[g] / wr[g]: pool blocks group g reads / writes; ws[g]: uses the workspace;
// coll[g]: a collective; active[g]: group takes part (incremental relaunch set).
// Returns the steps in issue order; a step with > 1 entries is a collective batch.
std::vector<std::vector<int>> collective_schedule(const std::vector<char>& active,
                                                  const std::vector<std::vector<int>>& rd,
                                                  const std::vector<std::vector<int>>& wr,
                                                  const std::vector<char>& ws,
                                                  const std::vector<char>& coll);

}  // namespace cg
