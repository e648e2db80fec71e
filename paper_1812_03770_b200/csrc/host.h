// Host compiler of the B200 computation-graph evaluator (no CUDA dependency).
//
// Implements, from the paper's text and the readings listed in DESIGN.md:
//   - the graph G = (V, E, lambda, U)                       [Def. 1, P:36-40]
//   - eager shape inference                                 [Shape layer, P:255-256]
//   - CSE -> constant folding -> DCE                        [Optimiser, P:264-272]
//   - post-order DFS ordering gamma                         [P:312; Def. 2, P:73-77]
//   - elementwise-chain fusion grouping                     [motivated by P:273, P:300]
//   - Algorithm 1 on groups (refcounts, FindBestBlock)      [P:292-364]
//   - canonical JSON dumps (compared byte-for-byte with the oracle's)
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/cg.h"

namespace cg {

using Shape = std::vector<int64_t>;

struct OpInfo {
  const char* name;
  int arity;  // -1 = variadic (>= 1)
  bool ew;    // elementwise (fusable, in-place safe)
  bool red;   // axis reduction (fusable as group sink)
  bool commutative;
};
const OpInfo& op_info(int op);
int64_t numel(const Shape& s);

struct Attr {
  int a0 = 0, a1 = 0, ta = 0, tb = 0, sh = 1, sw = 1, pad = 0, kh = 0, kw = 0, h = 0, w = 0, axis = 0;
  Shape dims;  // RESHAPE target
};

struct Node {
  int id = 0;
  int op = CG_VAR;
  std::vector<int> preds;
  Attr attr;
  Shape shape;
  std::vector<float> host;  // CONST data (VAR: optional initial value)
  bool raw_op = false;      // was an op node (not a leaf) when added: counts in unshared_bytes
  bool folded_pending = false;  // CF turned it into a CONST whose value the device has not produced yet
};

enum GroupKind { G_OP = 0, G_EW = 1, G_RED = 2 };

struct Group {
  int sink = -1;
  int kind = G_OP;
  bool has_domain = false;
  Shape domain;
  bool safe = false;
  std::vector<int> members;       // gamma order
  std::vector<int> inputs;        // distinct non-member values, by (member rank, slot)
  std::vector<int> materialised;  // sink + kept members, gamma order
};

struct Plan {
  // R14 zero-copy CONCAT views: node -> root (-1: not a view); element (o, i) of a
  // view is element o * view_inner_root + view_off + i of the root
  std::vector<int> view_root;
  std::vector<int64_t> view_outer, view_inner_root, view_off, view_inner;
  std::vector<int> block_of;         // node id -> block id (-1: not pooled)
  std::vector<uint64_t> size;        // block id -> bytes (exact, after growth)
  std::vector<uint64_t> offset;      // block id -> byte offset in the pool (256-aligned)
  uint64_t pool_bytes = 0, plan_bytes = 0;
};

struct Error {
  int code;
  std::string msg;
};

class HostGraph {
 public:
  // ---- build ----
  int add_node(int op, const int* inputs, int n, const cg_attr* a, Error* err);
  int add_update(int u, int var, Error* err);
  // ---- f1 pattern rewrites (cg_set_rewrites), applied at the start of optimise
  uint32_t rw_flags = 0;
  std::vector<int> rw_identity, rw_zeroed, rw_fma, rw_adagrad;
  void apply_rewrites(const std::vector<int>& outs, std::map<int, int>* rwrep);
  // ---- optimise (CSE -> CF -> DCE); returns the CF frontier whose values the device must produce
  int optimise(const std::vector<int>& outputs, cg_report* rep, std::vector<int>* frontier, Error* err);
  // rewrite the CF frontier into Consts (same id).  values[i] (may be empty in
  // host-only mode) is the device-computed value of folded[i].
  void apply_folds(const std::vector<std::vector<float>>& values);
  // ---- plan ----
  int plan(const std::vector<int>& outputs, uint32_t flags, Error* err);

  std::string graph_json() const;
  std::string plan_json() const;

  int resolve(int id) const {  // CSE representative
    auto it = rep.find(id);
    return it == rep.end() ? id : it->second;
  }
  bool is_external(int v) const { return nodes[v].op == CG_VAR || nodes[v].op == CG_CONST; }

  std::vector<Node> nodes;
  std::vector<std::pair<int, int>> updates;  // (source, Var), add order
  // optimise results
  bool optimised = false;
  std::vector<char> dead;
  std::vector<int> folded;
  std::map<int, int> rep;
  // plan results
  bool planned = false;
  uint32_t flags = 0;
  std::vector<int> outputs, roots, gamma, rank;  // rank: node -> gamma index (-1 if absent)
  std::vector<char> keep;                        // node -> kept (roots + incremental frontier)
  std::vector<Group> groups;                     // Gamma order
  std::vector<int> group_of;                     // node -> group index (-1 for leaves / absent)
  std::vector<std::vector<int>> desc_of_var;     // Var -> strict descendants in gamma (for dirtying)
  Plan pl;
  uint64_t unshared_bytes = 0;
};

std::string shape_str(const Shape& s);

}  // namespace cg
