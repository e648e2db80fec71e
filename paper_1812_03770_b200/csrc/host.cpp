#include <cstdlib>
// Host compiler: graph, shape inference, optimiser, ordering, fusion grouping,
// Algorithm 1 planner, canonical dumps.  See host.h for the paper anchors.
#include "host.h"

#include <algorithm>
#include <cstring>
#include <sstream>

namespace cg {

// ---------------------------------------------------------------- op table
// [Type layer, P:252-253]: operations as a variant type with fixed arities.
static const OpInfo kOps[CG_NUM_OPS] = {
    {"VAR", 0, false, false, false},          {"CONST", 0, false, false, false},
    {"ADD", 2, true, false, true},            {"SUB", 2, true, false, false},
    {"MUL", 2, true, false, true},            {"DIV", 2, true, false, false},
    {"POW", 2, true, false, false},           {"MAX2", 2, true, false, true},
    {"MIN2", 2, true, false, true},           {"RELU_GRAD", 2, true, false, false},
    {"FMA", 3, true, false, false},           {"NEG", 1, true, false, false},
    {"ABS", 1, true, false, false},           {"SQRT", 1, true, false, false},
    {"EXP", 1, true, false, false},           {"LOG", 1, true, false, false},
    {"SIN", 1, true, false, false},           {"COS", 1, true, false, false},
    {"TANH", 1, true, false, false},          {"RELU", 1, true, false, false},
    {"SUM", 1, false, true, false},           {"MAX", 1, false, true, false},
    {"DOT", 2, false, false, false},          {"CONV2D", 2, false, false, false},
    {"CONV2D_BWD_INPUT", 2, false, false, false}, {"CONV2D_BWD_KERNEL", 2, false, false, false},
    {"MAXPOOL2D", 1, false, false, false},    {"MAXPOOL2D_BWD", 2, false, false, false},
    {"AVGPOOL2D", 1, false, false, false},    {"CONCAT", -1, false, false, false},
    {"RESHAPE", 1, false, false, false},      {"ALLREDUCE_SUM", 1, false, false, false},
    {"FUSED_ADAGRAD", 4, true, false, false},
};

const OpInfo& op_info(int op) { return kOps[op]; }

int64_t numel(const Shape& s) {
  int64_t n = 1;
  for (auto d : s) n *= d;
  return n;
}

std::string shape_str(const Shape& s) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < s.size(); ++i) o << (i ? "," : "") << s[i];
  o << "]";
  return o.str();
}

// ---------------------------------------------------------------- shape inference
// [Shape layer, P:255-256]; rules in SURVEY §8(c) c1-defs and the padding convention.
static bool broadcast(const std::vector<const Shape*>& in, Shape* out) {
  size_t r = 0;
  for (auto* s : in) r = std::max(r, s->size());
  out->assign(r, 1);
  for (size_t k = 0; k < r; ++k) {
    int64_t e = 1;
    for (auto* s : in) {
      int64_t j = (int64_t)k - (int64_t)(r - s->size());
      if (j < 0) continue;
      int64_t d = (*s)[j];
      if (d == 1) continue;
      if (e == 1) e = d;
      else if (e != d) return false;
    }
    (*out)[k] = e;
  }
  return true;
}

static bool conv_out(int64_t in, int64_t k, int64_t s, int pad, int64_t* out) {
  if (s < 1 || k < 1) return false;
  if (pad == 1) { *out = (in + s - 1) / s; return true; }
  if (in < k) return false;
  *out = (in - k) / s + 1;
  return true;
}

static bool infer(int op, const std::vector<const Shape*>& in, const Attr& a, Shape* out, std::string* why) {
  const OpInfo& oi = op_info(op);
  if (oi.ew) {
    if (!broadcast(in, out)) { *why = "cannot broadcast operands"; return false; }
    return true;
  }
  switch (op) {
    case CG_SUM: case CG_MAX: {
      const Shape& x = *in[0];
      if (!(0 <= a.a0 && a.a0 < a.a1 && a.a1 <= (int)x.size())) { *why = "reduction axes out of range"; return false; }
      *out = x;
      for (int k = a.a0; k < a.a1; ++k) (*out)[k] = 1;
      return true;
    }
    case CG_DOT: {
      const Shape &A = *in[0], &B = *in[1];
      if (A.size() != 2 || B.size() != 2) { *why = "DOT needs rank-2 operands"; return false; }
      int64_t m = a.ta ? A[1] : A[0], k = a.ta ? A[0] : A[1];
      int64_t k2 = a.tb ? B[1] : B[0], n = a.tb ? B[0] : B[1];
      if (k != k2) { *why = "DOT inner dimensions differ"; return false; }
      *out = {m, n};
      return true;
    }
    case CG_CONV2D: {
      const Shape &x = *in[0], &w = *in[1];
      if (x.size() != 4 || w.size() != 4 || x[3] != w[2]) { *why = "CONV2D wants NHWC x HWIO with matching C"; return false; }
      int64_t ho, wo;
      if (!conv_out(x[1], w[0], a.sh, a.pad, &ho) || !conv_out(x[2], w[1], a.sw, a.pad, &wo)) { *why = "CONV2D window"; return false; }
      *out = {x[0], ho, wo, w[3]};
      return true;
    }
    case CG_CONV2D_BWD_INPUT: {
      const Shape &dy = *in[0], &w = *in[1];
      if (dy.size() != 4 || w.size() != 4 || dy[3] != w[3]) { *why = "CONV2D_BWD_INPUT operands"; return false; }
      int64_t ho, wo;
      if (!conv_out(a.h, w[0], a.sh, a.pad, &ho) || !conv_out(a.w, w[1], a.sw, a.pad, &wo) || ho != dy[1] || wo != dy[2]) {
        *why = "CONV2D_BWD_INPUT spatial mismatch"; return false;
      }
      *out = {dy[0], a.h, a.w, w[2]};
      return true;
    }
    case CG_CONV2D_BWD_KERNEL: {
      const Shape &x = *in[0], &dy = *in[1];
      if (x.size() != 4 || dy.size() != 4 || x[0] != dy[0]) { *why = "CONV2D_BWD_KERNEL operands"; return false; }
      int64_t ho, wo;
      if (!conv_out(x[1], a.kh, a.sh, a.pad, &ho) || !conv_out(x[2], a.kw, a.sw, a.pad, &wo) || ho != dy[1] || wo != dy[2]) {
        *why = "CONV2D_BWD_KERNEL spatial mismatch"; return false;
      }
      *out = {a.kh, a.kw, x[3], dy[3]};
      return true;
    }
    case CG_MAXPOOL2D: case CG_AVGPOOL2D: case CG_MAXPOOL2D_BWD: {
      const Shape& x = *in[0];
      if (x.size() != 4) { *why = "pool needs NHWC"; return false; }
      int64_t ho, wo;
      if (!conv_out(x[1], a.kh, a.sh, a.pad, &ho) || !conv_out(x[2], a.kw, a.sw, a.pad, &wo)) { *why = "pool window"; return false; }
      Shape py = {x[0], ho, wo, x[3]};
      if (op == CG_MAXPOOL2D_BWD) {
        if (*in[1] != py) { *why = "MAXPOOL2D_BWD dy shape mismatch"; return false; }
        *out = x;
      } else {
        *out = py;
      }
      return true;
    }
    case CG_CONCAT: {
      const Shape& s0 = *in[0];
      int r = (int)s0.size();
      if (a.axis < 0 || a.axis >= r) { *why = "CONCAT axis"; return false; }
      int64_t tot = 0;
      for (auto* s : in) {
        if ((int)s->size() != r) { *why = "CONCAT ranks"; return false; }
        for (int k = 0; k < r; ++k)
          if (k != a.axis && (*s)[k] != s0[k]) { *why = "CONCAT shapes"; return false; }
        tot += (*s)[a.axis];
      }
      *out = s0;
      (*out)[a.axis] = tot;
      return true;
    }
    case CG_RESHAPE: {
      for (auto d : a.dims)
        if (d < 1) { *why = "RESHAPE dims must be >= 1"; return false; }
      if (numel(a.dims) != numel(*in[0])) { *why = "RESHAPE changes element count"; return false; }
      *out = a.dims;
      return true;
    }
    case CG_ALLREDUCE_SUM:
      *out = *in[0];
      return true;
  }
  *why = "unknown op";
  return false;
}

static bool err_set(Error* e, int code, const std::string& msg) {
  if (e) { e->code = code; e->msg = msg; }
  return false;
}

// ---------------------------------------------------------------- build
int HostGraph::add_node(int op, const int* inputs, int n, const cg_attr* a, Error* err) {
  if (op < 0 || op >= CG_NUM_OPS) return err_set(err, CG_E_ARITY, "unknown op code"), CG_E_ARITY;
  const OpInfo& oi = op_info(op);
  int id = (int)nodes.size();
  if ((oi.arity >= 0 && n != oi.arity) || (oi.arity < 0 && n < 1)) {
    err_set(err, CG_E_ARITY, std::string("node ") + std::to_string(id) + ": " + oi.name + " takes " +
                                 std::to_string(oi.arity) + " inputs, got " + std::to_string(n));
    return CG_E_ARITY;
  }
  Node nd;
  nd.id = id;
  nd.op = op;
  if (op == CG_VAR || op == CG_CONST) {
    if (!a || a->ndim < 0 || a->ndim > 8) return err_set(err, CG_E_ARG, "leaf needs cg_attr with 0 <= ndim <= 8"), CG_E_ARG;
    for (int k = 0; k < a->ndim; ++k) {
      if (a->dims[k] < 1) return err_set(err, CG_E_SHAPE, "leaf extents must be >= 1"), CG_E_SHAPE;
      nd.shape.push_back(a->dims[k]);
    }
    if (op == CG_CONST && !a->host_data) return err_set(err, CG_E_ARG, "CONST needs host_data"), CG_E_ARG;
    if (a->host_data) nd.host.assign(a->host_data, a->host_data + numel(nd.shape));
    nodes.push_back(std::move(nd));
    return id;
  }
  std::vector<const Shape*> in;
  for (int k = 0; k < n; ++k) {
    if (inputs[k] < 0 || inputs[k] >= id) {
      err_set(err, CG_E_BAD_NODE, "node " + std::to_string(id) + ": unknown predecessor " + std::to_string(inputs[k]));
      return CG_E_BAD_NODE;
    }
    nd.preds.push_back(inputs[k]);
    in.push_back(&nodes[inputs[k]].shape);
  }
  cg_attr zero{};
  const cg_attr& A = a ? *a : zero;
  nd.attr.a0 = A.a0; nd.attr.a1 = A.a1; nd.attr.ta = A.ta ? 1 : 0; nd.attr.tb = A.tb ? 1 : 0;
  nd.attr.sh = A.sh; nd.attr.sw = A.sw; nd.attr.pad = A.pad ? 1 : 0;
  nd.attr.kh = A.kh; nd.attr.kw = A.kw; nd.attr.h = A.h; nd.attr.w = A.w; nd.attr.axis = A.axis;
  if (op == CG_RESHAPE) {
    if (A.ndim < 1 || A.ndim > 8) return err_set(err, CG_E_ARG, "RESHAPE needs 1 <= ndim <= 8"), CG_E_ARG;
    nd.attr.dims.assign(A.dims, A.dims + A.ndim);
  }
  std::string why;
  if (!infer(op, in, nd.attr, &nd.shape, &why)) {
    std::string ins;
    for (auto* s : in) ins += shape_str(*s);
    err_set(err, CG_E_SHAPE, "node " + std::to_string(id) + ": " + oi.name + " " + ins + ": " + why);
    return CG_E_SHAPE;
  }
  nd.raw_op = true;
  nodes.push_back(std::move(nd));
  return id;
}

int HostGraph::add_update(int u, int var, Error* err) {
  int n = (int)nodes.size();
  if (u < 0 || u >= n || var < 0 || var >= n) return err_set(err, CG_E_BAD_NODE, "update edge names an unknown node"), CG_E_BAD_NODE;
  if (nodes[var].op != CG_VAR)
    return err_set(err, CG_E_NOT_VAR, "update target " + std::to_string(var) + " is not a Var (Def. 1)"), CG_E_NOT_VAR;
  for (auto& e : updates)
    if (e.second == var) return err_set(err, CG_E_DUP_UPDATE, "Var " + std::to_string(var) + " already has an update edge"), CG_E_DUP_UPDATE;
  if (nodes[u].shape != nodes[var].shape)
    return err_set(err, CG_E_UPDATE_SHAPE, "update " + std::to_string(u) + "->" + std::to_string(var) + ": " +
                                               shape_str(nodes[u].shape) + " vs " + shape_str(nodes[var].shape)), CG_E_UPDATE_SHAPE;
  updates.emplace_back(u, var);
  return 0;
}

// ---------------------------------------------------------------- optimiser
// CSE (one ascending pass; commutative canonicalisation; Vars never merge;
// Consts merge by bytes; lowest id represents) -> CF (frontier folding) -> DCE.
static void put_i64(std::string& k, int64_t v) { k.append(reinterpret_cast<const char*>(&v), sizeof v); }

static std::string cse_key(const Node& n) {
  std::string k;
  put_i64(k, n.op);
  const Attr& a = n.attr;
  for (int v : {a.a0, a.a1, a.ta, a.tb, a.sh, a.sw, a.pad, a.kh, a.kw, a.h, a.w, a.axis}) put_i64(k, v);
  put_i64(k, (int64_t)a.dims.size());
  for (auto d : a.dims) put_i64(k, d);
  put_i64(k, (int64_t)n.shape.size());
  for (auto d : n.shape) put_i64(k, d);
  std::vector<int> p = n.preds;
  if (op_info(n.op).commutative) std::sort(p.begin(), p.end());
  put_i64(k, (int64_t)p.size());
  for (int q : p) put_i64(k, q);
  if (n.op == CG_CONST) k.append(reinterpret_cast<const char*>(n.host.data()), n.host.size() * sizeof(float));
  return k;
}

static void reach_back(const std::vector<Node>& nodes, const std::vector<int>& roots, std::vector<char>* live) {
  live->assign(nodes.size(), 0);
  std::vector<int> st(roots.begin(), roots.end());
  while (!st.empty()) {
    int v = st.back();
    st.pop_back();
    if ((*live)[v]) continue;
    (*live)[v] = 1;
    for (int p : nodes[v].preds) st.push_back(p);
  }
}

static void json_ints(std::ostringstream& o, const std::vector<int>& v);

// ---------------------------------------------------------------- pattern rewrites (f1)
// [Optimiser, P:273-279]; readings in DESIGN.md "f1 rewrites": ascending-id sweeps
// of identities, AdaGrad, FMA repeated to a fixpoint; keep nodes never removed or
// absorbed; "single consumer" = one consuming edge among live nodes.
static bool const_all(const Node& nd, float x) {
  if (nd.op != CG_CONST || nd.host.empty()) return false;
  for (float v : nd.host)
    if (!(v == x)) return false;
  return true;
}
static bool scalar_const(const Node& nd) {
  if (nd.op != CG_CONST) return false;
  for (auto d : nd.shape)
    if (d != 1) return false;
  return true;
}

void HostGraph::apply_rewrites(const std::vector<int>& outs, std::map<int, int>* rwrep) {
  const int n = (int)nodes.size();
  std::vector<char> keep(n, 0);
  for (int o : outs) keep[o] = 1;
  for (auto& e : updates) keep[e.first] = 1;
  auto res = [&](int v) {
    for (auto it = rwrep->find(v); it != rwrep->end(); it = rwrep->find(v)) v = it->second;
    return v;
  };
  auto redirect = [&]() {
    for (int v = 0; v < n; ++v)
      if (!dead[v])
        for (int& p : nodes[v].preds) p = res(p);
  };
  auto uses = [&]() {
    std::vector<int> u(n, 0);
    for (int v = 0; v < n; ++v)
      if (!dead[v])
        for (int p : nodes[v].preds) u[p]++;
    return u;
  };
  for (;;) {
    bool changed = false;
    if (rw_flags & CG_RW_IDENTITY) {
      redirect();
      for (int v = 0; v < n; ++v) {
        Node& nd = nodes[v];
        if (dead[v] || keep[v]) continue;
        if (nd.op != CG_ADD && nd.op != CG_SUB && nd.op != CG_MUL && nd.op != CG_DIV) continue;
        for (int& p : nd.preds) p = res(p);
        const int a = nd.preds[0], b = nd.preds[1];
        const bool sa = nodes[a].shape == nd.shape, sb = nodes[b].shape == nd.shape;
        int to = -1;
        if (nd.op == CG_ADD) {
          if (const_all(nodes[b], 0.f) && sa) to = a;
          else if (const_all(nodes[a], 0.f) && sb) to = b;
        } else if (nd.op == CG_SUB) {
          if (const_all(nodes[b], 0.f) && sa) to = a;
        } else if (nd.op == CG_MUL) {
          if (const_all(nodes[b], 1.f) && sa) to = a;
          else if (const_all(nodes[a], 1.f) && sb) to = b;
          else if (const_all(nodes[a], 0.f) || const_all(nodes[b], 0.f)) {
            nd.op = CG_CONST;
            nd.preds.clear();
            nd.attr = Attr();
            nd.host.assign((size_t)numel(nd.shape), 0.f);
            rw_zeroed.push_back(v);
            changed = true;
            continue;
          }
        } else if (nd.op == CG_DIV) {
          if (const_all(nodes[b], 1.f) && sa) to = a;
        }
        if (to >= 0) {
          (*rwrep)[v] = to;
          dead[v] = 1;
          rw_identity.push_back(v);
          changed = true;
        }
      }
    }
    if (rw_flags & CG_RW_ADAGRAD) {
      redirect();
      std::vector<int> cnt = uses();
      auto interior = [&](int v) { return !dead[v] && !keep[v] && cnt[v] == 1; };
      for (int v = 0; v < n; ++v) {
        Node& nd = nodes[v];
        if (dead[v] || nd.op != CG_DIV) continue;
        const int num = nd.preds[0], den = nd.preds[1];
        const Node &N = nodes[num], &D = nodes[den];
        if (N.op != CG_MUL || D.op != CG_ADD || !interior(num) || !interior(den)) continue;
        int lr, gg;
        if (scalar_const(nodes[N.preds[0]])) { lr = N.preds[0]; gg = N.preds[1]; }
        else if (scalar_const(nodes[N.preds[1]])) { lr = N.preds[1]; gg = N.preds[0]; }
        else continue;
        int q, eps;
        if (nodes[D.preds[0]].op == CG_SQRT && scalar_const(nodes[D.preds[1]])) { q = D.preds[0]; eps = D.preds[1]; }
        else if (nodes[D.preds[1]].op == CG_SQRT && scalar_const(nodes[D.preds[0]])) { q = D.preds[1]; eps = D.preds[0]; }
        else continue;
        if (!interior(q)) continue;
        const int sv = nodes[q].preds[0];
        nd.op = CG_FUSED_ADAGRAD;
        nd.preds = {gg, sv, lr, eps};
        dead[num] = dead[den] = dead[q] = 1;
        rw_adagrad.push_back(v);
        changed = true;
      }
    }
    if (rw_flags & CG_RW_FMA) {
      redirect();
      std::vector<int> cnt = uses();
      for (int v = 0; v < n; ++v) {
        Node& nd = nodes[v];
        if (dead[v] || nd.op != CG_ADD) continue;
        for (int side = 0; side < 2; ++side) {
          const int m = nd.preds[side], c = nd.preds[1 - side];
          if (nodes[m].op == CG_MUL && !dead[m] && !keep[m] && cnt[m] == 1) {
            const int a = nodes[m].preds[0], b = nodes[m].preds[1];
            nd.op = CG_FMA;
            nd.preds = {a, b, c};
            dead[m] = 1;
            rw_fma.push_back(v);
            changed = true;
            break;
          }
        }
      }
    }
    if (!changed) break;
  }
  redirect();
}

int HostGraph::optimise(const std::vector<int>& outs_raw, cg_report* report, std::vector<int>* frontier, Error* err) {
  int n = (int)nodes.size();
  for (int o : outs_raw)
    if (o < 0 || o >= n) return err_set(err, CG_E_BAD_NODE, "unknown output " + std::to_string(o)), CG_E_BAD_NODE;
  dead.assign(n, 0);
  rep.clear();
  folded.clear();
  rw_identity.clear(); rw_zeroed.clear(); rw_fma.clear(); rw_adagrad.clear();
  std::map<int, int> rwrep;
  if (rw_flags) apply_rewrites(outs_raw, &rwrep);
  auto rw = [&](int v) {
    for (auto it = rwrep.find(v); it != rwrep.end(); it = rwrep.find(v)) v = it->second;
    return v;
  };
  std::vector<int> outs_in;
  for (int o : outs_raw) outs_in.push_back(rw(o));
  for (auto& e : updates) e.first = rw(e.first);
  // CSE
  std::map<std::string, int> seen;
  for (int v = 0; v < n; ++v) {
    Node& nd = nodes[v];
    if (dead[v]) continue;  // removed by a rewrite
    for (int& p : nd.preds) p = resolve(p);
    if (nd.op == CG_VAR) continue;
    auto key = cse_key(nd);
    auto it = seen.find(key);
    if (it != seen.end()) {
      rep[v] = it->second;
      dead[v] = 1;
    } else {
      seen.emplace(std::move(key), v);
    }
  }
  std::vector<int> outs;
  for (int o : outs_in) outs.push_back(resolve(o));
  for (auto& e : updates) e.first = resolve(e.first);
  // every id removed by an identity rewrite resolves to its final representative
  for (auto& kv : rwrep) {
    const int t = rw(kv.first);
    rep[kv.first] = resolve(t);
  }
  std::vector<int> rts = outs;
  for (auto& e : updates) rts.push_back(e.first);
  // CF: C = Consts + non-(Var, ALLREDUCE) nodes with preds, all in C (ascending pass)
  std::vector<char> C(n, 0), isroot(n, 0);
  for (int r : rts) isroot[r] = 1;
  for (int v = 0; v < n; ++v) {
    if (dead[v]) continue;
    const Node& nd = nodes[v];
    if (nd.op == CG_CONST) { C[v] = 1; continue; }
    if (nd.op == CG_VAR || nd.op == CG_ALLREDUCE_SUM || nd.preds.empty()) continue;
    bool all = true;
    for (int p : nd.preds) all = all && C[p];
    C[v] = all;
  }
  std::vector<char> nonconst_consumer(n, 0);
  for (int v = 0; v < n; ++v) {
    if (dead[v]) continue;
    for (int p : nodes[v].preds)
      if (!C[v]) nonconst_consumer[p] = 1;
  }
  frontier->clear();
  for (int v = 0; v < n; ++v)
    if (C[v] && nodes[v].op != CG_CONST && (isroot[v] || nonconst_consumer[v])) frontier->push_back(v);
  // the caller evaluates the frontier's const cone on the device BEFORE we rewrite it;
  // here we only record the structural change (same id, op CONST, no preds)
  folded = *frontier;
  // DCE: keep what is reachable from the roots, treating folded nodes as leaves
  {
    std::vector<Node> view = nodes;
    for (int v : folded) view[v].preds.clear();
    std::vector<char> live;
    reach_back(view, rts, &live);
    int removed = 0;
    for (int v = 0; v < n; ++v)
      if (!dead[v] && nodes[v].op != CG_VAR && !live[v]) { dead[v] = 1; ++removed; }
    if (report) {
      report->cse_merged = (int)(rep.size() - rwrep.size());
      report->rw_identity = (int)rw_identity.size();
      report->rw_zeroed = (int)rw_zeroed.size();
      report->rw_fma = (int)rw_fma.size();
      report->rw_adagrad = (int)rw_adagrad.size();
      report->cf_folded = (int)folded.size();
      report->dce_removed = removed;
    }
  }
  optimised = true;
  return 0;
}

void HostGraph::apply_folds(const std::vector<std::vector<float>>& values) {
  for (size_t i = 0; i < folded.size(); ++i) {
    Node& nd = nodes[folded[i]];
    nd.op = CG_CONST;
    nd.preds.clear();
    nd.attr = Attr();
    if (i < values.size() && !values[i].empty()) {
      nd.host = values[i];
      nd.folded_pending = false;
    } else {
      nd.host.clear();
      nd.folded_pending = true;
    }
  }
}

// ---------------------------------------------------------------- ordering + grouping + plan
static std::vector<std::vector<int>> consumers(const std::vector<Node>& nodes, const std::vector<int>& order) {
  std::vector<std::vector<int>> cons(nodes.size());
  for (int v : order)
    for (int p : nodes[v].preds) {
      auto& c = cons[p];
      if (std::find(c.begin(), c.end(), v) == c.end()) c.push_back(v);
    }
  return cons;
}

namespace {
struct BlockSet {  // reusable blocks ordered by (size, id): O(log b) FindBestBlock [P:364]
  std::set<std::pair<uint64_t, int>> s;
};
}  // namespace

int HostGraph::plan(const std::vector<int>& outs_in, uint32_t fl, Error* err) {
  int n = (int)nodes.size();
  if (!optimised) dead.assign(n, 0);
  outputs.clear();
  for (int o : outs_in) {
    if (o < 0 || o >= n) return err_set(err, CG_E_BAD_NODE, "unknown output " + std::to_string(o)), CG_E_BAD_NODE;
    int r = resolve(o);
    if (dead[r]) return err_set(err, CG_E_BAD_NODE, "output " + std::to_string(o) + " was removed by cg_optimise"), CG_E_BAD_NODE;
    outputs.push_back(r);
  }
  flags = fl;
  const bool incremental = fl & CG_PLAN_INCREMENTAL, nofusion = fl & CG_PLAN_NO_FUSION;
  roots = outputs;
  for (auto& e : updates) roots.push_back(e.first);
  // gamma: iterative post-order DFS from the roots, preds left to right [P:312]
  gamma.clear();
  rank.assign(n, -1);
  {
    std::vector<char> seen(n, 0);
    for (int r : roots) {
      if (seen[r]) continue;
      seen[r] = 1;
      std::vector<std::pair<int, size_t>> st{{r, 0}};
      while (!st.empty()) {
        auto& top = st.back();
        const auto& pr = nodes[top.first].preds;
        if (top.second < pr.size()) {
          int p = pr[top.second++];
          if (!seen[p]) { seen[p] = 1; st.push_back({p, 0}); }
        } else {
          rank[top.first] = (int)gamma.size();
          gamma.push_back(top.first);
          st.pop_back();
        }
      }
    }
  }
  auto cons = consumers(nodes, gamma);
  // descendants of every Var (dirty propagation at run time and incremental signatures)
  desc_of_var.assign(n, {});
  std::vector<char> is_target(n, 0);
  for (auto& e : updates) is_target[e.second] = 1;
  std::vector<std::vector<int>> sig(n);
  keep.assign(n, 0);
  for (int r : roots) keep[r] = 1;
  for (int x : gamma) {
    if (nodes[x].op != CG_VAR) continue;
    std::vector<char> inD(n, 0);
    std::vector<int> st{x}, D;
    while (!st.empty()) {
      int v = st.back();
      st.pop_back();
      for (int c : cons[v])
        if (!inD[c]) { inD[c] = 1; D.push_back(c); st.push_back(c); }
    }
    std::sort(D.begin(), D.end(), [&](int a, int b) { return rank[a] < rank[b]; });
    desc_of_var[x] = D;
    if (is_target[x] || !incremental) continue;
    for (int v : D) sig[v].push_back(x);  // ascending x: sig vectors stay sorted
    for (int u : gamma) {                 // frontier F(x)
      if (u == x || inD[u]) continue;
      for (int c : cons[u])
        if (inD[c]) { keep[u] = 1; break; }
    }
  }
  // fusion grouping in reverse gamma
  groups.clear();
  group_of.assign(n, -1);
  std::vector<Group> rev;
  for (auto it = gamma.rbegin(); it != gamma.rend(); ++it) {
    int v = *it;
    const Node& nd = nodes[v];
    if (nd.op == CG_VAR || nd.op == CG_CONST) continue;
    const OpInfo& oi = op_info(nd.op);
    Group G;
    G.sink = v;
    G.members = {v};
    if (!oi.ew && !oi.red) {
      G.kind = G_OP;
    } else if (oi.red) {
      G.kind = G_RED;
      G.has_domain = true;
      G.domain = nodes[nd.preds[0]].shape;
    } else {
      std::vector<int> cg;
      for (int c : cons[v]) {
        int gi = group_of[c];
        if (std::find(cg.begin(), cg.end(), gi) == cg.end()) cg.push_back(gi);
      }
      if (cg.size() == 1 && !nofusion) {
        Group& T = rev[cg[0]];
        if (T.has_domain && nd.shape == T.domain && (!incremental || sig[v] == sig[T.sink])) {
          T.members.push_back(v);
          group_of[v] = cg[0];
          continue;
        }
      }
      G.kind = G_EW;
      G.has_domain = true;
      G.domain = nd.shape;
    }
    group_of[v] = (int)rev.size();
    rev.push_back(std::move(G));
  }
  std::vector<int> order(rev.size());
  for (size_t i = 0; i < rev.size(); ++i) order[i] = (int)i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return rank[rev[a].sink] < rank[rev[b].sink]; });
  std::vector<int> newidx(rev.size());
  for (size_t i = 0; i < order.size(); ++i) {
    newidx[order[i]] = (int)i;
    groups.push_back(std::move(rev[order[i]]));
  }
  for (int v : gamma)
    if (group_of[v] >= 0) group_of[v] = newidx[group_of[v]];
  for (auto& G : groups) {
    std::sort(G.members.begin(), G.members.end(), [&](int a, int b) { return rank[a] < rank[b]; });
    for (int m : G.members)
      for (int p : nodes[m].preds)
        if (group_of[p] != group_of[m] || is_external(p)) {
          if (std::find(G.inputs.begin(), G.inputs.end(), p) == G.inputs.end()) G.inputs.push_back(p);
        }
    for (int m : G.members)
      if (m == G.sink || keep[m]) G.materialised.push_back(m);
    bool allew = true;
    for (int m : G.members) allew = allew && op_info(nodes[m].op).ew;
    G.safe = allew || (G.members.size() == 1 &&
                       (nodes[G.sink].op == CG_RESHAPE || nodes[G.sink].op == CG_ALLREDUCE_SUM));
  }
  // Algorithm 1 on groups [P:323-362] with readings R1-R14
  pl = Plan();
  pl.block_of.assign(n, -1);
  std::vector<int> refs(n, 0);
  for (auto& G : groups)
    for (int p : G.inputs)
      if (!is_external(p)) refs[p]++;
  // R14 zero-copy CONCAT: inputs planned as views of the concat's block (outer
  // concats first, so nested concats map to one root); see oracle/planner.py
  pl.view_root.assign(n, -1);
  pl.view_outer.assign(n, 0);
  pl.view_inner_root.assign(n, 0);
  pl.view_off.assign(n, 0);
  pl.view_inner.assign(n, 0);
  if (!incremental && !getenv("CG_NO_CONCAT_VIEWS")) {  // (the env switch is a debugging aid: dumps then differ)
    std::vector<char> is_sink(n, 0);
    std::vector<int> consumers(n, 0);
    for (auto& G : groups) {
      is_sink[G.sink] = 1;
      for (int p : G.inputs) consumers[p]++;
    }
    for (auto it = groups.rbegin(); it != groups.rend(); ++it) {
      const int c = it->sink;
      const Node& nc = nodes[c];
      if (nc.op != CG_CONCAT) continue;
      const int ax = nc.attr.axis;
      int64_t outer = 1, inner_c = 1;
      for (int k = 0; k < (int)nc.shape.size(); ++k) (k < ax ? outer : inner_c) *= nc.shape[k];
      int root = c;
      int64_t inner_root = inner_c, base = 0;
      if (pl.view_root[c] >= 0) {
        if (pl.view_outer[c] != outer) continue;
        root = pl.view_root[c];
        inner_root = pl.view_inner_root[c];
        base = pl.view_off[c];
      }
      int64_t off = 0;
      for (int v : nc.preds) {
        int64_t inner_v = 1;
        for (int k = ax; k < (int)nodes[v].shape.size(); ++k) inner_v *= nodes[v].shape[k];
        const int op = nodes[v].op;
        const bool once = std::count(nc.preds.begin(), nc.preds.end(), v) == 1;
        if (is_sink[v] && !is_external(v) && op != CG_RESHAPE && op != CG_ALLREDUCE_SUM && !keep[v] &&
            consumers[v] == 1 && once) {
          pl.view_root[v] = root;
          pl.view_outer[v] = outer;
          pl.view_inner_root[v] = inner_root;
          pl.view_off[v] = base + off;
          pl.view_inner[v] = inner_v;
        }
        off += inner_v;
      }
    }
  }
  std::set<std::pair<uint64_t, int>> reusable;
  auto& size = pl.size;
  auto new_block = [&](uint64_t s) {
    size.push_back(s);
    return (int)size.size() - 1;
  };
  auto find_best_block = [&](uint64_t s, const std::vector<int>& pref) -> int {
    auto lb = reusable.lower_bound({s, -1});
    if (lb != reusable.end()) {
      std::pair<uint64_t, int> best = *lb;
      bool have_pref = false;
      for (int b : pref) {  // in-place preference restricted to sufficient blocks (R5)
        std::pair<uint64_t, int> c{size[b], b};
        if (size[b] < s || !reusable.count(c)) continue;
        if (!have_pref || c < best) { best = c; have_pref = true; }
      }
      reusable.erase(best);
      return best.second;
    }
    if (!reusable.empty()) {  // grow the largest reusable block, lowest id on ties (R1, R8)
      uint64_t smax = reusable.rbegin()->first;
      auto it = reusable.lower_bound({smax, -1});
      int b = it->second;
      reusable.erase(it);
      size[b] = s;
      return b;
    }
    return new_block(s);
  };
  for (auto& G : groups) {
    std::vector<int> released;
    auto release = [&](bool phase_filter, bool want_full) {
      int64_t dn = numel(nodes[G.sink].shape);
      for (int p : G.inputs) {
        if (is_external(p)) continue;
        if (phase_filter && ((numel(nodes[p].shape) == dn) != want_full)) continue;
        if (--refs[p] == 0 && !keep[p] && pl.view_root[p] < 0) {
          reusable.insert({size[pl.block_of[p]], pl.block_of[p]});
          released.push_back(p);
        }
      }
    };
    if (G.safe) release(true, true);
    for (int m : G.materialised) {
      uint64_t nb = 4 * (uint64_t)numel(nodes[m].shape);
      if (pl.view_root[m] >= 0 || pl.block_of[m] >= 0) {  // R14: the family's root block
        const int root = pl.view_root[m] >= 0 ? pl.view_root[m] : m;
        if (pl.block_of[root] < 0) pl.block_of[root] = find_best_block(4 * (uint64_t)numel(nodes[root].shape), {});
        pl.block_of[m] = pl.block_of[root];
      } else if (incremental && keep[m]) {
        pl.block_of[m] = new_block(nb);
      } else {
        std::vector<int> pref;
        for (int p : released)
          if (numel(nodes[p].shape) == numel(nodes[m].shape)) pref.push_back(pl.block_of[p]);
        pl.block_of[m] = find_best_block(nb, pref);
      }
    }
    if (G.safe) release(true, false);
    else release(false, false);
  }
  uint64_t off = 0;
  pl.offset.clear();
  for (auto s : size) {
    pl.offset.push_back(off);
    off += (s + 255) / 256 * 256;
    pl.plan_bytes += s;
  }
  pl.pool_bytes = off;
  unshared_bytes = 0;
  for (auto& nd : nodes)
    if (nd.raw_op) unshared_bytes += 4 * (uint64_t)numel(nd.shape);
  planned = true;
  return 0;
}

// ---------------------------------------------------------------- dumps
static void json_ints(std::ostringstream& o, const std::vector<int>& v) {
  o << "[";
  for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
  o << "]";
}

static void json_attrs(std::ostringstream& o, const Node& nd) {
  const Attr& a = nd.attr;
  o << "{";
  switch (nd.op) {
    case CG_SUM: case CG_MAX: o << "\"a0\":" << a.a0 << ",\"a1\":" << a.a1; break;
    case CG_DOT: o << "\"ta\":" << a.ta << ",\"tb\":" << a.tb; break;
    case CG_CONV2D: o << "\"pad\":" << a.pad << ",\"sh\":" << a.sh << ",\"sw\":" << a.sw; break;
    case CG_CONV2D_BWD_INPUT:
      o << "\"h\":" << a.h << ",\"pad\":" << a.pad << ",\"sh\":" << a.sh << ",\"sw\":" << a.sw << ",\"w\":" << a.w;
      break;
    case CG_CONV2D_BWD_KERNEL: case CG_MAXPOOL2D: case CG_MAXPOOL2D_BWD: case CG_AVGPOOL2D:
      o << "\"kh\":" << a.kh << ",\"kw\":" << a.kw << ",\"pad\":" << a.pad << ",\"sh\":" << a.sh << ",\"sw\":" << a.sw;
      break;
    case CG_CONCAT: o << "\"axis\":" << a.axis; break;
    case CG_RESHAPE: {
      o << "\"dims\":[";
      for (size_t i = 0; i < a.dims.size(); ++i) o << (i ? "," : "") << a.dims[i];
      o << "]";
      break;
    }
    default: break;
  }
  o << "}";
}

std::string HostGraph::graph_json() const {
  std::ostringstream o;
  std::vector<int> dd;
  for (size_t v = 0; v < dead.size(); ++v)
    if (dead[v]) dd.push_back((int)v);
  std::vector<int> fo = folded;
  std::sort(fo.begin(), fo.end());
  o << "{\"dead\":";
  json_ints(o, dd);
  o << ",\"folded\":";
  json_ints(o, fo);
  o << ",\"nodes\":[";
  bool first = true;
  for (const auto& nd : nodes) {
    if (!dead.empty() && dead[nd.id]) continue;
    o << (first ? "" : ",") << "{\"attrs\":";
    first = false;
    json_attrs(o, nd);
    o << ",\"id\":" << nd.id << ",\"op\":\"" << op_info(nd.op).name << "\",\"preds\":";
    json_ints(o, nd.preds);
    o << ",\"shape\":[";
    for (size_t i = 0; i < nd.shape.size(); ++i) o << (i ? "," : "") << nd.shape[i];
    o << "]}";
  }
  o << "],\"rep\":[";
  first = true;
  for (auto& kv : rep) {
    o << (first ? "" : ",") << "[" << kv.first << "," << kv.second << "]";
    first = false;
  }
  o << "]";
  if (rw_flags) {
    auto srt = [](std::vector<int> v) { std::sort(v.begin(), v.end()); return v; };
    o << ",\"rewrites\":{\"adagrad\":";
    json_ints(o, srt(rw_adagrad));
    o << ",\"fma\":";
    json_ints(o, srt(rw_fma));
    o << ",\"identity\":";
    json_ints(o, srt(rw_identity));
    o << ",\"zeroed\":";
    json_ints(o, srt(rw_zeroed));
    o << "}";
  }
  o << "}";
  return o.str();
}

std::string HostGraph::plan_json() const {
  std::ostringstream o;
  o << "{\"block\":[";
  bool first = true;
  for (size_t v = 0; v < pl.block_of.size(); ++v)
    if (pl.block_of[v] >= 0) {
      o << (first ? "" : ",") << "[" << v << "," << pl.block_of[v] << "]";
      first = false;
    }
  o << "],\"block_bytes\":[";
  for (size_t b = 0; b < pl.size.size(); ++b) o << (b ? "," : "") << pl.size[b];
  o << "],\"gamma\":";
  json_ints(o, gamma);
  o << ",\"groups\":[";
  for (size_t i = 0; i < groups.size(); ++i) {
    const Group& G = groups[i];
    o << (i ? "," : "") << "{\"inputs\":";
    json_ints(o, G.inputs);
    o << ",\"materialised\":";
    json_ints(o, G.materialised);
    o << ",\"members\":";
    json_ints(o, G.members);
    o << ",\"sink\":" << G.sink << "}";
  }
  o << "],\"keep\":[";
  first = true;
  for (int v = 0; v < (int)keep.size(); ++v)
    if (keep[v] && rank[v] >= 0 && !is_external(v)) {
      o << (first ? "" : ",") << v;
      first = false;
    }
  o << "],\"plan_bytes\":" << pl.plan_bytes << ",\"pool_bytes\":" << pl.pool_bytes
    << ",\"unshared_bytes\":" << unshared_bytes << ",\"views\":[";
  first = true;
  for (int v = 0; v < (int)pl.view_root.size(); ++v)
    if (pl.view_root[v] >= 0) {
      o << (first ? "" : ",") << "[" << v << "," << pl.view_root[v] << "," << pl.view_outer[v] << ","
        << pl.view_inner_root[v] << "," << pl.view_off[v] << "," << pl.view_inner[v] << "]";
      first = false;
    }
  o << "]}";
  return o.str();
}

}  // namespace cg
