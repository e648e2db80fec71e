// Code generator for fused groups.  Every member op rounds to fp32 exactly as
// the eager definition does (IEEE __fadd_rn/__fmul_rn/__fdiv_rn/__fsqrt_rn, no
// contraction; NVRTC also gets --fmad=false), so fusion changes memory traffic,
// never values [fusion "to reduce memory access", P:273].
//
// Elementwise groups ("ew"): the group domain is collapsed (adjacent dims merge
// when every operand's strides allow it), then one of two thread mappings:
//   row  : domain viewed as [R, W]; 128-bit vector loads along W; operands that
//          do not depend on the row (row-broadcast, scalars) are loaded once per
//          thread before the row loop; column-broadcast operands are one load per
//          row; 2 rows per thread per iteration for memory-level parallelism.
//   flat : vector index over the whole domain; contiguous operands use 128-bit
//          loads, broadcast operands index by compile-time div/mod.
// Reduction groups ("red"): domain [O, Rn, I] (axes before / inside / after
// [a0, a1)); thread block = TX (over I, coalesced) x TY (over Rn) x TO (over O);
// each thread accumulates sequentially, then a fixed-order shared-memory tree
// over TY; large Rn is split over grid.z into workspace partials reduced by a
// second fixed-order kernel.  No atomics: results are run-to-run bit-stable.
#include "codegen.h"

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <functional>
#include <map>
#include <sstream>

namespace cg {

namespace {

Shape contiguous_strides(const Shape& s) {
  Shape st(s.size(), 1);
  for (int k = (int)s.size() - 2; k >= 0; --k) st[k] = st[k + 1] * s[k + 1];
  return st;
}

// stride of `op` (broadcast to `dom`, numpy trailing alignment) along each domain dim
Shape bstrides(const Shape& op, const Shape& dom) {
  Shape cs = contiguous_strides(op);
  Shape out(dom.size(), 0);
  int r = (int)dom.size(), ro = (int)op.size();
  for (int k = 0; k < r; ++k) {
    int j = k - (r - ro);
    if (j >= 0 && op[j] != 1) out[k] = cs[j];
  }
  return out;
}

std::string expr(int op, const std::vector<std::string>& a) {
  switch (op) {
    case CG_ADD: return "__fadd_rn(" + a[0] + "," + a[1] + ")";
    case CG_SUB: return "__fsub_rn(" + a[0] + "," + a[1] + ")";
    case CG_MUL: return "__fmul_rn(" + a[0] + "," + a[1] + ")";
    case CG_DIV: return "__fdiv_rn(" + a[0] + "," + a[1] + ")";
    case CG_POW: return "powf(" + a[0] + "," + a[1] + ")";
    case CG_MAX2: return "cg_max(" + a[0] + "," + a[1] + ")";
    case CG_MIN2: return "cg_min(" + a[0] + "," + a[1] + ")";
    case CG_RELU_GRAD: return "(" + a[0] + " > 0.f ? " + a[1] + " : 0.f)";
    case CG_FMA: return "__fmaf_rn(" + a[0] + "," + a[1] + "," + a[2] + ")";
    case CG_NEG: return "(-" + a[0] + ")";
    case CG_ABS: return "fabsf(" + a[0] + ")";
    case CG_SQRT: return "__fsqrt_rn(" + a[0] + ")";
    case CG_EXP: {
      // CG_FAST_EXP=1 (measurement only): 2^(x log2 e) on the SFU, see cg_exp2e
      static const bool fast = getenv("CG_FAST_EXP") && atoi(getenv("CG_FAST_EXP")) == 1;
      return (fast ? "cg_exp2e(" : "expf(") + a[0] + ")";
    }
    case CG_LOG: return "logf(" + a[0] + ")";
    case CG_SIN: return "sinf(" + a[0] + ")";
    case CG_COS: return "cosf(" + a[0] + ")";
    case CG_TANH: return "tanhf(" + a[0] + ")";
    case CG_RELU: return "(" + a[0] + " > 0.f ? " + a[0] + " : 0.f)";
    case CG_FUSED_ADAGRAD:  // lr*g / (sqrt(s) + eps) in f64, one rounding (the oracle's definition)
      return "((float)((double)" + a[2] + " * (double)" + a[0] + " / (sqrt((double)" + a[1] + ") + (double)" + a[3] + ")))";
  }
  return "0.f";
}

const char* kPrelude = R"(
typedef unsigned long long u64;
// CG_FAST_EXP=1 only (measurement, not the default): exp(x) = 2^RN(x log2 e) on the
// SFU, relative error <= |x| 2^-23 + 2 ulp (libm expf: <= 2 ulp).  C2 under the power
// cap: 90-94 % -> 96.5-97 % of HBM (its chain is issue-bound there; a compensated
// 2.5-ulp variant with four more instructions measured no gain), so the default stays
// the accurate expf.
__device__ __forceinline__ float cg_exp2e(float x) {
  float r;
  asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(__fmul_rn(x, 1.44269504088896341f)));
  return r;
}
__device__ __forceinline__ float4 cg_ld4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void cg_st4(float* p, float a, float b, float c, float d) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
// NaN-propagating max/min (numpy maximum/minimum, the oracle's definition)
__device__ __forceinline__ float cg_max(float a, float b) {
  float r; asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ float cg_min(float a, float b) {
  float r; asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ float cg_lane(const float4& v, int l) {
  return l == 0 ? v.x : (l == 1 ? v.y : (l == 2 ? v.z : v.w));
}
)";

uint64_t fnv(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) { h ^= c; h *= 0x100000001b3ULL; }
  return h;
}

thread_local std::string g_helpers;  // device helpers of the kernel being generated

std::string finish(const std::string& kind, const std::string& body_with_KNAME, std::string* name) {
  char buf[64];
  snprintf(buf, sizeof buf, "cg_%s_%016llx", kind.c_str(), (unsigned long long)fnv(body_with_KNAME));
  *name = buf;
  std::string src = body_with_KNAME;
  size_t pos;
  while ((pos = src.find("KNAME")) != std::string::npos) src.replace(pos, 5, *name);
  return std::string(kPrelude) + g_helpers + src;
}

// Collapse domain dims: drop extent-1 dims, merge adjacent dims when every operand allows.
void collapse(const Shape& dom, std::vector<Shape>& strides, Shape* ext_out) {
  Shape ext;
  std::vector<Shape> st(strides.size());
  for (size_t k = 0; k < dom.size(); ++k) {
    if (dom[k] == 1) continue;
    ext.push_back(dom[k]);
    for (size_t o = 0; o < strides.size(); ++o) st[o].push_back(strides[o][k]);
  }
  // merge from the inside out
  for (int k = (int)ext.size() - 2; k >= 0; --k) {
    bool ok = true;
    for (auto& s : st) ok = ok && (s[k] == s[k + 1] * ext[k + 1]);
    if (!ok) continue;
    ext[k] *= ext[k + 1];
    ext.erase(ext.begin() + k + 1);
    for (auto& s : st) { s[k] = s[k + 1]; s.erase(s.begin() + k + 1); }
  }
  if (ext.empty()) {
    ext.push_back(1);
    for (auto& s : st) s.push_back(0);
  }
  *ext_out = ext;
  strides = st;
}

std::string i64(int64_t v) { return std::to_string(v) + "LL"; }

// Offset of an operand with collapsed ext/strides at flat index e, as a device
// helper with compile-time div/mod (appended to `helpers`); returns the call.
std::string offset_expr(const std::string& e, const Shape& ext, const Shape& st, const std::string& itype,
                        std::string* helpers) {
  int k = (int)ext.size();
  int jmin = -1;
  for (int j = 0; j < k; ++j)
    if (st[j] != 0) { jmin = j; break; }
  if (jmin < 0) return "0";
  std::ostringstream o;
  o << "{ " << itype << " q_ = e_; " << itype << " off_ = 0; ";
  for (int j = k - 1; j > jmin; --j) {
    o << "off_ += (q_ % (" << itype << ")" << ext[j] << ") * (" << itype << ")" << st[j] << "; q_ /= (" << itype << ")"
      << ext[j] << "; ";
  }
  // dims outside jmin have stride 0, so the coordinate of jmin is q_ mod its extent
  if (jmin > 0) o << "off_ += (q_ % (" << itype << ")" << ext[jmin] << ") * (" << itype << ")" << st[jmin] << "; ";
  else o << "off_ += q_ * (" << itype << ")" << st[jmin] << "; ";
  o << "return off_; }";
  std::string body = o.str();
  char nm[40];
  snprintf(nm, sizeof nm, "cg_off_%016llx", (unsigned long long)fnv(body + itype));
  std::string def = "__device__ __forceinline__ " + itype + " " + nm + "(" + itype + " e_) " + body + "\n";
  if (helpers->find(def) == std::string::npos) *helpers += def;
  return std::string(nm) + "((" + itype + ")(" + e + "))";
}

struct MemberEmitter {
  const HostGraph& hg;
  const Group& G;
  // value name of node p for lane l: input k -> x<k>_<l>, member m -> v<m>_<l>
  std::function<std::string(int, int)> name;
  std::string emit(int lanes) const {
    std::ostringstream o;
    for (int l = 0; l < lanes; ++l)
      for (int m : G.members) {
        const Node& nd = hg.nodes[m];
        if (op_info(nd.op).red) continue;
        std::vector<std::string> a;
        for (int p : nd.preds) a.push_back(name(p, l));
        o << "      const float v" << m << "_" << l << " = " << expr(nd.op, a) << ";\n";
      }
    return o.str();
  }
};

int input_index(const Group& G, int p) {
  for (size_t k = 0; k < G.inputs.size(); ++k)
    if (G.inputs[k] == p) return (int)k;
  return -1;
}

std::string args_decl(const Group& G, const std::vector<int>& outs, bool ws) {
  std::ostringstream o;
  bool first = true;
  for (size_t k = 0; k < G.inputs.size(); ++k) {
    o << (first ? "" : ", ") << "const float* __restrict__ in" << k;
    first = false;
  }
  for (size_t j = 0; j < outs.size(); ++j) {
    o << (first ? "" : ", ") << "float* __restrict__ out" << j;
    first = false;
  }
  if (ws) o << (first ? "" : ", ") << "float* __restrict__ ws";
  return o.str();
}

// ------------------------------------------------------------------ elementwise
KernelSpec gen_ew(const HostGraph& hg, const Group& G, int num_sms) {
  KernelSpec ks;
  const Shape& dom = G.domain;
  const int64_t N = numel(dom);
  ks.in_ids = G.inputs;
  ks.out_ids = G.materialised;
  const size_t nin = G.inputs.size(), nout = G.materialised.size();
  std::vector<Shape> st;
  for (int p : G.inputs) st.push_back(bstrides(hg.nodes[p].shape, dom));
  for (size_t j = 0; j < nout; ++j) st.push_back(contiguous_strides(dom));
  Shape ext;
  collapse(dom, st, &ext);
  int k = (int)ext.size();
  int64_t W = ext[k - 1];
  bool inner_ok = true;
  for (size_t q = 0; q < nin; ++q) inner_ok = inner_ok && (st[q][k - 1] == 0 || st[q][k - 1] == 1);
  const int V = (W % 4 == 0 && inner_ok) ? 4 : 1;
  const std::string itype = N < (1LL << 31) ? "unsigned" : "u64";
  MemberEmitter me{hg, G, [&](int p, int l) {
                     int q = input_index(G, p);
                     if (q >= 0) return "x" + std::to_string(q) + "_" + std::to_string(l);
                     return "v" + std::to_string(p) + "_" + std::to_string(l);
                   }};
  std::ostringstream b;
  // ---- row mode ----
  int64_t R = 1;
  std::vector<int64_t> so(nin), si(nin);
  bool row = false;
  // row mode needs a 2-D view whose rows are short enough to unroll (KC <= 8 column
  // chunks per thread) and numerous enough to fill the grid; a fully collapsed 1-D
  // domain (only full-size and scalar operands) is exactly the flat mode's case.
  if (k == 2 && W / V >= 32 && (W / V + 255) / 256 <= 8) {
    R = ext[0];
    for (size_t q = 0; q < nin; ++q) {
      si[q] = st[q][1];
      so[q] = st[q][0];
    }
    row = true;
  }
  // rows (row mode) / vectors (flat mode) in flight per thread per iteration;
  // CG_EW_UNROLL overrides for measurement sweeps
  // (measured on C2, tools/ew_sweep.sh: row mode 1 row -> 6.68 TB/s, 2 -> 6.09, 4 -> 6.60)
  static const int U_env = getenv("CG_EW_UNROLL") ? atoi(getenv("CG_EW_UNROLL")) : 0;
  const int U_row = U_env > 0 ? U_env : 1;
  const int U = U_env > 0 ? U_env : 2;
  if (row) {
    ks.mode = "row";
    const int64_t WV = W / V;
    int TX = (int)std::min<int64_t>(256, (WV + 31) / 32 * 32);
    int TY = 256 / TX;
    // block = exactly TX x TY threads: a thread with ty >= TY would revisit rows of
    // the next block, which in an in-place (slid) group reads already-written output
    ks.block = (uint32_t)(TX * TY);
    int KC = (int)((WV + TX - 1) / TX);
    bool hoist = KC <= 4;
    b << "extern \"C\" __global__ void __launch_bounds__(" << TX * TY << ") KNAME(" << args_decl(G, G.materialised, false)
      << ") {\n";
    b << "  const int tx = threadIdx.x % " << TX << ", ty = threadIdx.x / " << TX << ";\n";
    // hoisted operands (do not depend on the row)
    for (size_t q = 0; q < nin; ++q) {
      if (so[q] != 0) continue;
      if (si[q] == 0) {
        b << "  const float h" << q << " = in" << q << "[0];\n";
      } else if (hoist) {
        for (int j = 0; j < KC; ++j) {
          b << "  float4 h" << q << "_" << j << " = make_float4(0.f,0.f,0.f,0.f);\n";
          b << "  if (tx + " << j * TX << " < " << WV << ") ";
          if (V == 4) b << "h" << q << "_" << j << " = cg_ld4(in" << q << " + (tx + " << j * TX << ") * 4);\n";
          else b << "h" << q << "_" << j << ".x = in" << q << "[(tx + " << j * TX << ") * " << si[q] << "];\n";
        }
      }
    }
    // software-pipelined variant (1 row per iteration, CG_EW_PREFETCH=1): the next
    // row's loads are issued before this row's arithmetic.  Measured on C2 under
    // sw_power_cap (tools/ew_prefetch_ab.sh, 3 interleaved pairs): 5,700 GB/s vs
    // 5,930 without -- occupancy already hides the latency and the extra live
    // registers cost more -- so it is off by default.
    static const bool prefetch = getenv("CG_EW_PREFETCH") && atoi(getenv("CG_EW_PREFETCH")) == 1;
    if (prefetch && U_row == 1) {
      auto is_rowdep = [&](size_t q) { return !(so[q] == 0 && (si[q] == 0 || hoist)); };
      b << "  const long long step = (long long)gridDim.x * " << TY << ";\n";
      b << "  long long rb = (long long)blockIdx.x * " << TY << " + ty;\n";
      for (int j = 0; j < KC; ++j)
        for (size_t q = 0; q < nin; ++q) {
          if (!is_rowdep(q)) continue;
          if (si[q] != 0 && V == 4) b << "  float4 p" << q << "_" << j << " = make_float4(0.f,0.f,0.f,0.f);\n";
          else b << "  float p" << q << "_" << j << " = 0.f;\n";
        }
      auto emit_loads = [&](const std::string& rv, const std::string& ind) {
        for (int j = 0; j < KC; ++j) {
          b << ind << "{ const int c = tx + " << j * TX << "; if (c < " << WV << ") {\n";
          for (size_t q = 0; q < nin; ++q) {
            if (!is_rowdep(q)) continue;
            if (si[q] == 0) b << ind << " p" << q << "_" << j << " = in" << q << "[" << rv << " * " << so[q] << "LL];\n";
            else if (V == 4) b << ind << " p" << q << "_" << j << " = cg_ld4(in" << q << " + " << rv << " * " << so[q] << "LL + c * 4);\n";
            else b << ind << " p" << q << "_" << j << " = in" << q << "[" << rv << " * " << so[q] << "LL + c * " << si[q] << "LL];\n";
          }
          b << ind << "} }\n";
        }
      };
      b << "  if (rb < " << R << "LL) {\n";
      emit_loads("rb", "   ");
      b << "  }\n";
      b << "  for (; rb < " << R << "LL; rb += step) {\n";
      b << "   const long long rn = rb + step;\n";
      for (int j = 0; j < KC; ++j) {
        b << "   {\n    const int c = tx + " << j * TX << ";\n";
        b << "    if (c < " << WV << ") {\n";
        for (size_t q = 0; q < nin; ++q) {
          if (!is_rowdep(q)) continue;
          if (si[q] != 0 && V == 4) b << "     const float4 f" << q << "_0 = p" << q << "_" << j << ";\n";
          else b << "     const float s" << q << "_0 = p" << q << "_" << j << ";\n";
        }
        b << "     if (rn < " << R << "LL) {\n";
        for (size_t q = 0; q < nin; ++q) {
          if (!is_rowdep(q)) continue;
          if (si[q] == 0) b << "      p" << q << "_" << j << " = in" << q << "[rn * " << so[q] << "LL];\n";
          else if (V == 4) b << "      p" << q << "_" << j << " = cg_ld4(in" << q << " + rn * " << so[q] << "LL + c * 4);\n";
          else b << "      p" << q << "_" << j << " = in" << q << "[rn * " << so[q] << "LL + c * " << si[q] << "LL];\n";
        }
        b << "     }\n     {\n";
        for (int l = 0; l < V; ++l)
          for (size_t q = 0; q < nin; ++q) {
            b << "      const float x" << q << "_" << l << " = ";
            if (so[q] == 0 && si[q] == 0) b << "h" << q;
            else if (so[q] == 0 && hoist) b << (V == 4 ? "cg_lane(h" : "(h") << q << "_" << j << (V == 4 ? ", " + std::to_string(l) + ")" : ".x)");
            else if (si[q] == 0) b << "s" << q << "_0";
            else if (V == 4) b << "cg_lane(f" << q << "_0, " << l << ")";
            else b << "s" << q << "_0";
            b << ";\n";
          }
        b << me.emit(V);
        for (size_t jo = 0; jo < nout; ++jo) {
          int m = G.materialised[jo];
          if (V == 4)
            b << "      cg_st4(out" << jo << " + rb * " << W << "LL + c * 4, v" << m << "_0, v" << m << "_1, v" << m << "_2, v" << m
              << "_3);\n";
          else
            b << "      out" << jo << "[rb * " << W << "LL + c] = v" << m << "_0;\n";
        }
        b << "     }\n    }\n   }\n";
      }
      b << "  }\n}\n";
      int64_t work = (R + TY - 1) / TY;
      ks.work_blocks = work;
      ks.grid[0] = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(work, (int64_t)num_sms * 8));
      ks.source = finish("ew", b.str(), &ks.name);
      return ks;
    }
    b << "  const long long step = (long long)gridDim.x * " << TY * U_row << ";\n";
    b << "  for (long long rb = (long long)blockIdx.x * " << TY * U_row << " + ty; rb < " << R << "LL; rb += step) {\n";
    for (int j = 0; j < KC; ++j) {
      b << "   {\n    const int c = tx + " << j * TX << ";\n";
      b << "    if (c < " << WV << ") {\n";
      for (int u = 0; u < U_row; ++u) {
        b << "     const long long r" << u << " = rb + " << u * TY << ";\n";
        b << "     const bool ok" << u << " = r" << u << " < " << R << "LL;\n";
      }
      // loads for all U_row rows first (memory-level parallelism)
      for (int u = 0; u < U_row; ++u) {
        for (size_t q = 0; q < nin; ++q) {
          std::string rv = "r" + std::to_string(u);
          if (so[q] == 0 && (si[q] == 0 || hoist)) continue;
          if (si[q] == 0) {
            b << "     const float s" << q << "_" << u << " = ok" << u << " ? in" << q << "[" << rv << " * " << so[q] << "LL] : 0.f;\n";
          } else if (V == 4) {
            b << "     const float4 f" << q << "_" << u << " = ok" << u << " ? cg_ld4(in" << q << " + " << rv << " * " << so[q]
              << "LL + c * 4) : make_float4(0.f,0.f,0.f,0.f);\n";
          } else {
            b << "     const float s" << q << "_" << u << " = ok" << u << " ? in" << q << "[" << rv << " * " << so[q] << "LL + c * "
              << si[q] << "LL] : 0.f;\n";
          }
        }
      }
      for (int u = 0; u < U_row; ++u) {
        b << "     {\n";
        for (int l = 0; l < V; ++l)
          for (size_t q = 0; q < nin; ++q) {
            b << "      const float x" << q << "_" << l << " = ";
            if (so[q] == 0 && si[q] == 0) b << "h" << q;
            else if (so[q] == 0 && hoist) b << (V == 4 ? "cg_lane(h" : "(h") << q << "_" << j << (V == 4 ? ", " + std::to_string(l) + ")" : ".x)");
            else if (si[q] == 0) b << "s" << q << "_" << u;
            else if (V == 4) b << "cg_lane(f" << q << "_" << u << ", " << l << ")";
            else b << "s" << q << "_" << u;
            b << ";\n";
          }
        b << me.emit(V);
        b << "      if (ok" << u << ") {\n";
        for (size_t jo = 0; jo < nout; ++jo) {
          int m = G.materialised[jo];
          if (V == 4)
            b << "       cg_st4(out" << jo << " + r" << u << " * " << W << "LL + c * 4, v" << m << "_0, v" << m << "_1, v" << m
              << "_2, v" << m << "_3);\n";
          else
            b << "       out" << jo << "[r" << u << " * " << W << "LL + c] = v" << m << "_0;\n";
        }
        b << "      }\n     }\n";
      }
      b << "    }\n   }\n";
    }
    b << "  }\n}\n";
    int64_t work = (R + TY * U_row - 1) / (TY * U_row);
    ks.work_blocks = work;
    ks.grid[0] = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(work, (int64_t)num_sms * 8));
    ks.source = finish("ew", b.str(), &ks.name);
    return ks;
  }
  // ---- flat mode ----
  ks.mode = "flat";
  const int64_t NV = N / V;
  std::vector<int> kind(nin);  // 0 full-contiguous, 1 scalar, 2 general
  Shape cst = contiguous_strides(ext);
  for (size_t q = 0; q < nin; ++q) {
    bool zero = true, full = true;
    for (int j = 0; j < k; ++j) {
      zero = zero && st[q][j] == 0;
      full = full && st[q][j] == cst[j];
    }
    kind[q] = full ? 0 : (zero ? 1 : 2);
  }
  b << "extern \"C\" __global__ void __launch_bounds__(256) KNAME(" << args_decl(G, G.materialised, false) << ") {\n";
  for (size_t q = 0; q < nin; ++q)
    if (kind[q] == 1) b << "  const float h" << q << " = in" << q << "[0];\n";
  b << "  const " << itype << " step = (" << itype << ")gridDim.x * " << 256 * U << ";\n";
  b << "  for (" << itype << " t0 = (" << itype << ")blockIdx.x * " << 256 * U << " + threadIdx.x; t0 < (" << itype << ")" << NV
    << "; t0 += step) {\n";
  for (int u = 0; u < U; ++u) {
    b << "   const " << itype << " t" << u + 1 << " = t0 + " << 256 * u << ";\n";
    b << "   const bool ok" << u << " = t" << u + 1 << " < (" << itype << ")" << NV << ";\n";
    b << "   const " << itype << " e" << u << " = (ok" << u << " ? t" << u + 1 << " : 0) * " << V << ";\n";
  }
  for (int u = 0; u < U; ++u)
    for (size_t q = 0; q < nin; ++q) {
      if (kind[q] == 0) {
        if (V == 4) b << "   const float4 f" << q << "_" << u << " = cg_ld4(in" << q << " + e" << u << ");\n";
        else b << "   const float s" << q << "_" << u << "_0 = in" << q << "[e" << u << "];\n";
      } else if (kind[q] == 2) {
        for (int l = 0; l < V; ++l)
          b << "   const float s" << q << "_" << u << "_" << l << " = in" << q << "["
            << offset_expr("e" + std::to_string(u) + " + " + std::to_string(l), ext, st[q], itype, &g_helpers) << "];\n";
      }
    }
  for (int u = 0; u < U; ++u) {
    b << "   {\n";
    for (int l = 0; l < V; ++l)
      for (size_t q = 0; q < nin; ++q) {
        b << "    const float x" << q << "_" << l << " = ";
        if (kind[q] == 1) b << "h" << q;
        else if (kind[q] == 0 && V == 4) b << "cg_lane(f" << q << "_" << u << ", " << l << ")";
        else b << "s" << q << "_" << u << "_" << l;
        b << ";\n";
      }
    b << me.emit(V);
    b << "    if (ok" << u << ") {\n";
    for (size_t jo = 0; jo < nout; ++jo) {
      int m = G.materialised[jo];
      if (V == 4)
        b << "     cg_st4(out" << jo << " + e" << u << ", v" << m << "_0, v" << m << "_1, v" << m << "_2, v" << m << "_3);\n";
      else
        b << "     out" << jo << "[e" << u << "] = v" << m << "_0;\n";
    }
    b << "    }\n   }\n";
  }
  b << "  }\n}\n";
  int64_t work = (NV + 256 * U - 1) / (256 * U);
  ks.work_blocks = work;
  ks.grid[0] = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(work, (int64_t)num_sms * 8));
  ks.source = finish("ew", b.str(), &ks.name);
  return ks;
}

// ------------------------------------------------------------------ reduction
struct Seg {  // one of the O / R / I segments of the domain for one operand
  bool simple;
  int64_t stride;               // when simple
  Shape ext, st;                // when not simple (dims of the segment with extent > 1)
};

Seg make_seg(const Shape& dom, const Shape& s, int lo, int hi) {
  Seg g;
  for (int k = lo; k < hi; ++k)
    if (dom[k] != 1) { g.ext.push_back(dom[k]); g.st.push_back(s[k]); }
  g.simple = true;
  for (size_t j = 0; j + 1 < g.ext.size(); ++j)
    if (g.st[j] != g.st[j + 1] * g.ext[j + 1]) g.simple = false;
  g.stride = g.ext.empty() ? 0 : g.st.back();
  if (!g.ext.empty() && g.simple) {
    // an all-broadcast segment has stride 0 everywhere
    bool allz = true;
    for (auto v : g.st) allz = allz && v == 0;
    if (allz) g.stride = 0;
  }
  return g;
}

std::string seg_off(const Seg& g, const std::string& idx) {
  if (g.simple) return g.stride ? "(" + idx + ") * " + i64(g.stride) : "0LL";
  return offset_expr(idx, g.ext, g.st, "long long", &g_helpers);
}

KernelSpec gen_red(const HostGraph& hg, const Group& G, int num_sms) {
  KernelSpec ks;
  ks.mode = "red";
  const Node& sink = hg.nodes[G.sink];
  const Shape& dom = G.domain;
  const int a0 = sink.attr.a0, a1 = sink.attr.a1, r = (int)dom.size();
  int64_t O = 1, Rn = 1, I = 1;
  for (int kk = 0; kk < a0; ++kk) O *= dom[kk];
  for (int kk = a0; kk < a1; ++kk) Rn *= dom[kk];
  for (int kk = a1; kk < r; ++kk) I *= dom[kk];
  ks.in_ids = G.inputs;
  std::vector<int> interior;
  for (int m : G.materialised)
    if (m != G.sink) interior.push_back(m);
  ks.out_ids = interior;
  ks.out_ids.push_back(G.sink);
  ks.red_op = sink.op;
  ks.red_out = G.sink;
  const size_t nin = G.inputs.size();
  // launch geometry
  int TX = (int)std::min<int64_t>(I, 256);
  int TYmax = 256 / TX;
  int TY = 1;
  while (TY * 2 <= TYmax && TY < Rn) TY *= 2;
  int TO = (int)std::max<int64_t>(1, std::min<int64_t>(O, 256 / (TX * TY)));
  int64_t bx = (I + TX - 1) / TX, by = (O + TO - 1) / TO;
  int64_t blocks = bx * by;
  int64_t S = 1;
  // split the reduced extent until ~8 blocks per SM are in flight (each thread then
  // walks >= 16 rows: a short chain of dependent load batches) -- C3's bias gradients
  // [4096, 1024] -> [1, 1024]: 4 x 74 blocks -> 4 x 256
  if (blocks < 8LL * num_sms && Rn > 16LL * TY) {
    S = std::min<int64_t>((8LL * num_sms + blocks - 1) / blocks, Rn / (16LL * TY));
    S = std::max<int64_t>(1, std::min<int64_t>(S, 65535));
  }
  int64_t CH = (Rn + S - 1) / S;
  S = (Rn + CH - 1) / CH;
  ks.splits = S;
  ks.oi = O * I;
  ks.uses_ws = S > 1;
  ks.ws_floats = S > 1 ? (uint64_t)(S * O * I) : 0;
  ks.grid[0] = (uint32_t)bx;
  ks.grid[1] = (uint32_t)std::min<int64_t>(by, 65535);
  ks.grid[2] = (uint32_t)S;
  ks.block = TX * TY * TO;
  const int P = [&] { int p = 1; while (p * 2 <= TY) p *= 2; return p; }();
  const bool is_sum = sink.op == CG_SUM;
  const std::string ident = is_sum ? "0.f" : "(-__int_as_float(0x7f800000))";
  auto comb = [&](const std::string& a, const std::string& bb) {
    return is_sum ? "__fadd_rn(" + a + ", " + bb + ")" : "cg_max(" + a + ", " + bb + ")";
  };
  std::vector<Seg> sO, sR, sI;
  for (int p : G.inputs) {
    Shape s = bstrides(hg.nodes[p].shape, dom);
    sO.push_back(make_seg(dom, s, 0, a0));
    sR.push_back(make_seg(dom, s, a0, a1));
    sI.push_back(make_seg(dom, s, a1, r));
  }
  MemberEmitter me{hg, G, [&](int p, int l) {
                     int q = input_index(G, p);
                     if (q >= 0) return "x" + std::to_string(q) + "_" + std::to_string(l);
                     return "v" + std::to_string(p) + "_" + std::to_string(l);
                   }};
  int red_in = sink.preds[0];
  std::string red_val = me.name(red_in, 0);
  std::ostringstream b;
  b << "extern \"C\" __global__ void __launch_bounds__(" << ks.block << ") KNAME(" << args_decl(G, ks.out_ids, ks.uses_ws)
    << ") {\n";
  b << "  __shared__ float sm[" << ks.block << "];\n";
  b << "  const int tx = threadIdx.x % " << TX << ", ty = (threadIdx.x / " << TX << ") % " << TY << ", to = threadIdx.x / "
    << TX * TY << ";\n";
  b << "  const long long i = (long long)blockIdx.x * " << TX << " + tx;\n";
  b << "  const long long r_lo = (long long)blockIdx.z * " << CH << "LL;\n";
  b << "  const long long r_hi = min(r_lo + " << CH << "LL, " << Rn << "LL);\n";
  b << "  for (long long ob = blockIdx.y; ob < " << by << "LL; ob += gridDim.y) {\n";
  b << "   const long long o = ob * " << TO << " + to;\n";
  b << "   float acc = " << ident << ";\n";
  b << "   if (i < " << I << "LL && o < " << O << "LL) {\n";
  // hoisted: inputs whose R segment is simple with stride 0
  std::vector<bool> hoisted(nin, false);
  for (size_t q = 0; q < nin; ++q) {
    if (sR[q].simple && sR[q].stride == 0) {
      hoisted[q] = true;
      b << "    const float x" << q << "_0 = in" << q << "[" << seg_off(sO[q], "o") << " + " << seg_off(sI[q], "i") << "];\n";
    }
  }
  // main loop: RU consecutive rows of this thread per iteration, all loads first
  // (memory-level parallelism), then the prologue ops and the accumulation in
  // row order -- the same summation order as one row at a time
  const int RU = 4;
  b << "    long long rr = r_lo + ty;\n";
  b << "    for (; rr + " << (RU - 1) * TY << " < r_hi; rr += " << RU * TY << ") {\n";
  for (size_t q = 0; q < nin; ++q)
    for (int l = 0; l < RU; ++l) {
      if (hoisted[q]) {
        if (l) b << "     const float x" << q << "_" << l << " = x" << q << "_0;\n";
        continue;
      }
      b << "     const float x" << q << "_" << l << " = in" << q << "[" << seg_off(sO[q], "o") << " + "
        << seg_off(sR[q], "rr + " + std::to_string(l * TY)) << " + " << seg_off(sI[q], "i") << "];\n";
    }
  b << me.emit(RU);
  for (int l = 0; l < RU; ++l) {
    for (size_t j = 0; j < interior.size(); ++j)
      b << "     out" << j << "[(o * " << Rn << "LL + rr + " << l * TY << ") * " << I << "LL + i] = v" << interior[j] << "_" << l
        << ";\n";
    b << "     acc = " << comb("acc", me.name(red_in, l)) << ";\n";
  }
  b << "    }\n";
  b << "    for (; rr < r_hi; rr += " << TY << ") {\n";
  for (size_t q = 0; q < nin; ++q) {
    if (hoisted[q]) continue;
    b << "     const float x" << q << "_0 = in" << q << "[" << seg_off(sO[q], "o") << " + " << seg_off(sR[q], "rr") << " + "
      << seg_off(sI[q], "i") << "];\n";
  }
  b << me.emit(1);
  for (size_t j = 0; j < interior.size(); ++j)
    b << "     out" << j << "[(o * " << Rn << "LL + rr) * " << I << "LL + i] = v" << interior[j] << "_0;\n";
  b << "     acc = " << comb("acc", red_val) << ";\n";
  b << "    }\n   }\n";
  // fixed-order block tree over ty
  b << "   sm[threadIdx.x] = acc;\n   __syncthreads();\n";
  if (TY > P) {
    b << "   if (ty >= " << P << ") { const int d = threadIdx.x - " << P * TX << "; sm[d] = " << comb("sm[d]", "sm[threadIdx.x]")
      << "; }\n   __syncthreads();\n";
  }
  for (int h = P / 2; h >= 1; h /= 2) {
    b << "   if (ty < " << h << ") sm[threadIdx.x] = " << comb("sm[threadIdx.x]", "sm[threadIdx.x + " + std::to_string(h * TX) + "]")
      << ";\n   __syncthreads();\n";
  }
  b << "   if (ty == 0 && i < " << I << "LL && o < " << O << "LL) ";
  int oj = (int)interior.size();
  if (ks.uses_ws) b << "ws[((long long)blockIdx.z * " << O << "LL + o) * " << I << "LL + i] = sm[threadIdx.x];\n";
  else b << "out" << oj << "[o * " << I << "LL + i] = sm[threadIdx.x];\n";
  b << "   __syncthreads();\n";
  b << "  }\n}\n";
  ks.source = finish("red", b.str(), &ks.name);
  return ks;
}

}  // namespace

// ------------------------------------------------------------------ row runs
// Reduce -> broadcast fusion across groups ("single-kernel
// softmax"): a run of consecutive EW / row-reduction groups over a [B, N] domain
// (reductions over axis 1 only, N <= 1024) is one kernel with a warp per row.
// Each group's members are evaluated in Gamma order with the row's values in
// registers (lane l holds columns l, l+32, ...); a row reduction is a lane-local
// sequential pass then a fixed xor-butterfly (deterministic); every materialised
// value of every group is stored exactly as the group's own kernel would store it.
// Returns an empty name when the run does not qualify.
KernelSpec gen_rowrun(const HostGraph& hg, const std::vector<const Group*>& run, int num_sms) {
  g_helpers.clear();
  KernelSpec ks;
  if (run.size() < 2) return ks;
  int64_t B = -1, N = -1;
  for (const Group* G : run) {
    if (G->kind != G_EW && G->kind != G_RED) return ks;
    const Shape& d = G->domain;
    if (d.size() != 2) return ks;
    if (B < 0) B = d[0];
    if (d[0] != B) return ks;
    if (G->kind == G_RED) {
      const Node& sk = hg.nodes[G->sink];
      if ((sk.op != CG_SUM && sk.op != CG_MAX) || sk.attr.a0 != 1 || sk.attr.a1 != 2 || d[1] < 1) return ks;
      if (N < 0) N = d[1];
      if (d[1] != N) return ks;
    } else if (d[1] != 1) {
      if (N < 0) N = d[1];
      if (d[1] != N) return ks;
    }
  }
  if (N < 1 || N > 1024 || B < 1) return ks;
  const int NT = (int)((N + 31) / 32);
  // values produced inside the run: array ([B, N]) or row scalar ([B, 1])
  std::map<int, bool> made;  // node -> is array
  std::vector<int> ext;      // external inputs, first-use order
  std::map<int, int> ext_kind;  // 0 full [B,N], 1 row [B,1], 2 column [N], 3 scalar
  auto kind_of = [&](int p) -> int {
    const Shape& s = hg.nodes[p].shape;
    const int64_t n = numel(s);
    if (n == 1) return 3;
    if (s.size() == 2 && s[0] == B && s[1] == N) return 0;
    if (s.size() == 2 && s[0] == B && s[1] == 1) return 1;
    if ((s.size() == 2 && s[0] == 1 && s[1] == N) || (s.size() == 1 && s[0] == N)) return 2;
    return -1;
  };
  for (const Group* G : run)
    for (int m : G->members) {
      const Node& nd = hg.nodes[m];
      for (int p : nd.preds) {
        if (made.count(p) || ext_kind.count(p)) continue;
        const int k = kind_of(p);
        if (k < 0) return ks;
        ext_kind[p] = k;
        ext.push_back(p);
      }
      const bool arr = nd.shape.size() == 2 && nd.shape[1] == N && N > 1 ? true : (nd.shape.size() == 2 && nd.shape[1] == 1 ? false : N == 1);
      if (op_info(nd.op).red) {
        if (m != G->sink) return ks;
        made[m] = false;
      } else {
        if (!(nd.shape.size() == 2 && nd.shape[0] == B && (nd.shape[1] == N || nd.shape[1] == 1))) return ks;
        made[m] = arr;
      }
    }
  std::vector<int> outs;
  for (const Group* G : run)
    for (int m : G->materialised) outs.push_back(m);
  ks.in_ids = ext;
  ks.out_ids = outs;
  ks.mode = "rowrun";
  std::ostringstream b;
  b << "extern \"C\" __global__ void __launch_bounds__(256) KNAME(";
  for (size_t q = 0; q < ext.size(); ++q) b << (q ? ", " : "") << "const float* __restrict__ in" << q;
  for (size_t j = 0; j < outs.size(); ++j) b << ", float* __restrict__ out" << j;
  b << ") {\n";
  b << "  const int lane = threadIdx.x & 31;\n";
  b << "  for (long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); r < " << B << "LL; r += (long long)gridDim.x * 8) {\n";
  // externals: full / column operands loaded once per row (per t), row / scalar once
  auto name = [&](int p, const std::string& t) -> std::string {
    auto it = made.find(p);
    if (it != made.end()) return it->second ? "v" + std::to_string(p) + "[" + t + "]" : "v" + std::to_string(p);
    const int q = (int)(std::find(ext.begin(), ext.end(), p) - ext.begin());
    const int k = ext_kind[p];
    return (k == 0 || k == 2) ? "x" + std::to_string(q) + "[" + t + "]" : "x" + std::to_string(q);
  };
  for (size_t q = 0; q < ext.size(); ++q) {
    const int k = ext_kind[ext[q]];
    if (k == 0 || k == 2) {
      b << "   float x" << q << "[" << NT << "];\n";
      b << "#pragma unroll\n   for (int t = 0; t < " << NT << "; ++t) { const int j = lane + 32 * t; x" << q << "[t] = j < " << N
        << " ? in" << q << "[" << (k == 0 ? "r * " + std::to_string(N) + "LL + j" : std::string("j")) << "] : 0.f; }\n";
    } else {
      b << "   const float x" << q << " = in" << q << "[" << (k == 1 ? "r" : "0") << "];\n";
    }
  }
  for (const Group* G : run) {
    for (int m : G->members) {
      const Node& nd = hg.nodes[m];
      if (op_info(nd.op).red) {
        const int src = nd.preds[0];
        const bool sum = nd.op == CG_SUM;
        b << "   float v" << m << " = " << (sum ? "0.f" : "__int_as_float(0xff800000)") << ";\n";
        b << "#pragma unroll\n   for (int t = 0; t < " << NT << "; ++t) if (lane + 32 * t < " << N << ") v" << m << " = "
          << (sum ? "__fadd_rn(v" : "cg_max(v") << m << ", " << name(src, "t") << ");\n";
        b << "#pragma unroll\n   for (int o = 16; o > 0; o >>= 1) { const float y = __shfl_xor_sync(0xffffffffu, v" << m
          << ", o); v" << m << " = " << (sum ? "__fadd_rn(v" : "cg_max(v") << m << ", y); }\n";
        continue;
      }
      if (made[m]) {
        b << "   float v" << m << "[" << NT << "];\n";
        b << "#pragma unroll\n   for (int t = 0; t < " << NT << "; ++t) {\n";
        std::vector<std::string> a;
        for (int p : nd.preds) a.push_back(name(p, "t"));
        b << "    v" << m << "[t] = " << expr(nd.op, a) << ";\n   }\n";
      } else {
        std::vector<std::string> a;
        for (int p : nd.preds) a.push_back(name(p, "0"));
        b << "   const float v" << m << " = " << expr(nd.op, a) << ";\n";
      }
    }
  }
  for (size_t jo = 0; jo < outs.size(); ++jo) {
    const int m = outs[jo];
    if (made[m])
      b << "#pragma unroll\n   for (int t = 0; t < " << NT << "; ++t) { const int j = lane + 32 * t; if (j < " << N << ") out" << jo
        << "[r * " << N << "LL + j] = v" << m << "[t]; }\n";
    else
      b << "   if (lane == 0) out" << jo << "[r] = v" << m << ";\n";
  }
  b << "  }\n}\n";
  ks.block = 256;
  ks.work_blocks = (B + 7) / 8;
  ks.grid[0] = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(ks.work_blocks, (int64_t)num_sms * 8));
  ks.source = finish("run", b.str(), &ks.name);
  return ks;
}

KernelSpec gen_group(const HostGraph& hg, const Group& G, int num_sms) {
  g_helpers.clear();
  if (G.kind == G_RED) return gen_red(hg, G, num_sms);
  return gen_ew(hg, G, num_sms);
}

}  // namespace cg
