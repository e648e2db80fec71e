"""Pins of the oracle against what the paper and the mathematics fix (CPU only).

Each test names the passage (P:n = PAPER.md, S:n = SPEC.md) or the closed
form it checks.  None of these re-types an oracle formula: values come from
the paper's worked examples, hand traces, brute-force loops or identities.
"""
import math

import numpy as np
import pytest

from oracle import ops
from oracle.dump import compile_graph, graph_json, plan_json
from oracle.eager import evaluate, leaf_values, run_iterations
from oracle.graph import Graph, from_spec
from oracle.ops import CGError
from oracle.planner import find_best_block
from oracle.schedule import FLAG_INCREMENTAL, FLAG_NO_FUSION, gamma
from oracle.validate import validate_plan
from workloads import configs, gen


# ---------------------------------------------------------------- generator
def test_generator_known_values():
    # splitmix64 reference output for state 0 and FNV-1a-64 reference values
    assert gen.splitmix64_int(0) == 0xE220A8397B1DCDAF
    assert gen.fnv1a64("") == 0xCBF29CE484222325
    assert gen.fnv1a64("a") == 0xAF63DC4C8601EC8C
    a = gen.materialise({"kind": "uniform", "tag": "t", "lo": 0, "hi": 1}, [64, 8])
    b = gen.materialise({"kind": "uniform", "tag": "t", "lo": 0, "hi": 1}, [64, 8], rows=[3, 17])
    c = gen.materialise({"kind": "uniform", "tag": "t", "lo": 0, "hi": 1}, [32, 8], row_offset=32)
    assert np.array_equal(a[[3, 17]], b) and np.array_equal(a[32:], c)
    assert a.min() >= 0 and a.max() < 1
    # 24-bit grid: u * 2^24 is an integer
    assert np.all(np.floor(a.astype(np.float64) * 2**24) == a.astype(np.float64) * 2**24)


# ---------------------------------------------------------------- Fig. 1
def _fig1():
    g, outs = from_spec(configs.c1(4))
    return g, outs


def test_fig1_structure_and_gamma():
    g, outs = _fig1()
    assert [n.op for n in g.nodes] == ["CONST", "VAR", "SUB", "VAR", "MUL", "SIN"]
    edges = sorted((p, n.id) for n in g.nodes for p in n.preds)
    assert edges == [(0, 2), (1, 2), (2, 4), (3, 4), (4, 5)]  # 5 edges
    # post-order DFS from x5 gives the easypebbling labels 0..5
    assert gamma(g, outs) == [0, 1, 2, 3, 4, 5]


def test_fig1_values():
    g, outs = _fig1()
    v = evaluate(g, leaf_values(g, {1: np.full(4, 2.0), 3: np.full(4, 5.0)}))
    assert np.all(v[5] == 0) and np.all(v[2] == 0)  # x1 = 2 -> all-zero tail
    v = evaluate(g, leaf_values(g, {1: np.full(4, 1.0), 3: np.full(4, 0.5)}))
    assert np.all(v[5] == np.float32(math.sin(0.5)))  # sin((2-1)*0.5)


def test_counter_update_edge_three_rounds():
    # c' = c + 1 with iopair (c', c), c = 0: three rounds -> 3
    g = Graph()
    c = g.add_leaf("VAR", [1], data={"kind": "zeros"})
    one = g.add_leaf("CONST", [], data={"kind": "literal", "values": [1.0]})
    c1 = g.add_node("ADD", [c, one])
    g.add_update(c1, c)
    hist, state = run_iterations(g, [c1], 3)
    assert [float(h[c1][0]) for h in hist] == [1.0, 2.0, 3.0]
    assert float(state[c][0]) == 3.0


def test_add_node_errors():
    g = Graph()
    x = g.add_leaf("VAR", [2, 3])
    y = g.add_leaf("VAR", [3, 2])
    with pytest.raises(CGError) as e:
        g.add_node("ADD", [x])
    assert e.value.code == "CG_E_ARITY"
    with pytest.raises(CGError) as e:
        g.add_node("NEG", [7])
    assert e.value.code == "CG_E_BAD_NODE"
    with pytest.raises(CGError) as e:
        g.add_node("ADD", [x, y])
    assert e.value.code == "CG_E_SHAPE"
    m = g.add_node("NEG", [x])
    with pytest.raises(CGError) as e:
        g.add_update(x, m)
    assert e.value.code == "CG_E_NOT_VAR"  # Def. 1: lambda(v) = Var
    with pytest.raises(CGError) as e:
        g.add_update(m, y)
    assert e.value.code == "CG_E_UPDATE_SHAPE"
    g.add_update(m, x)
    with pytest.raises(CGError) as e:
        g.add_update(m, x)
    assert e.value.code == "CG_E_DUP_UPDATE"


def test_shape_rules():
    assert ops.broadcast_shape((3, 1), (1, 4)) == (3, 4)
    assert ops.broadcast_shape((5,), (5,)) == (5,)
    with pytest.raises(CGError):
        ops.broadcast_shape((2, 3), (4, 3))
    assert ops.infer_shape("DOT", [(2, 3), (3, 4)], {"ta": 0, "tb": 0}) == (2, 4)
    assert ops.infer_shape("DOT", [(3, 2), (4, 3)], {"ta": 1, "tb": 1}) == (2, 4)
    assert ops.infer_shape("RESHAPE", [(6,)], {"dims": [2, 3]}) == (2, 3)
    with pytest.raises(CGError):
        ops.infer_shape("RESHAPE", [(6,)], {"dims": [4, 2]})
    assert ops.infer_shape("SUM", [(4, 5, 6)], {"a0": 1, "a1": 3}) == (4, 1, 1)
    conv = lambda x, w, s, p: ops.infer_shape("CONV2D", [x, w], {"sh": s, "sw": s, "pad": p})
    assert conv((8, 28, 28, 1), (5, 5, 1, 6), 1, 1) == (8, 28, 28, 6)    # LeNet conv1 SAME
    assert conv((8, 14, 14, 6), (5, 5, 6, 16), 1, 0) == (8, 10, 10, 16)  # conv2 VALID
    assert conv((1, 299, 299, 3), (3, 3, 3, 32), 2, 0) == (1, 149, 149, 32)  # Inception stem
    assert ops.infer_shape("MAXPOOL2D", [(1, 147, 147, 64)],
                           {"kh": 3, "kw": 3, "sh": 2, "sw": 2, "pad": 0}) == (1, 73, 73, 64)


# ---------------------------------------------------------------- optimiser
def test_constant_folding_examples():
    # Const(2) - Const(1) feeding Mul(., Var x) -> Const(1) feeding Mul
    g = Graph()
    a = g.add_leaf("CONST", [], data={"kind": "literal", "values": [2.0]})
    b = g.add_leaf("CONST", [], data={"kind": "literal", "values": [1.0]})
    x = g.add_leaf("VAR", [3])
    d = g.add_node("SUB", [a, b])
    m = g.add_node("MUL", [d, x])
    c = compile_graph(g, [m])
    assert c.opt.folded == [d] and c.g.nodes[d].op == "CONST" and float(c.g.nodes[d].value) == 1.0
    assert {k: c.opt.report[k] for k in ("cse_merged", "cf_folded", "dce_removed")} == {"cse_merged": 0, "cf_folded": 1, "dce_removed": 2}
    # all-const graph -> a single Const
    g = Graph()
    a = g.add_leaf("CONST", [2], data={"kind": "literal", "values": [1.0, 2.0]})
    e = g.add_node("EXP", [a])
    s = g.add_node("ADD", [e, a])
    c = compile_graph(g, [s])
    live_ops = [c.g.nodes[i].op for i in c.opt.live()]
    assert live_ops == ["CONST"] and c.opt.folded == [s]
    assert np.allclose(c.g.nodes[s].value, np.exp([1.0, 2.0]) + [1.0, 2.0], rtol=1e-7)
    # Fig. 1 unchanged
    g, outs = _fig1()
    c = compile_graph(g, outs)
    assert {k: c.opt.report[k] for k in ("cse_merged", "cf_folded", "dce_removed")} == {"cse_merged": 0, "cf_folded": 0, "dce_removed": 0}


def test_cse_rules():
    g = Graph()
    x = g.add_leaf("VAR", [4])
    y = g.add_leaf("VAR", [4])
    x2 = g.add_leaf("VAR", [4])      # Vars never merge
    k1 = g.add_leaf("CONST", [], data={"kind": "literal", "values": [3.0]})
    k2 = g.add_leaf("CONST", [], data={"kind": "literal", "values": [3.0]})  # equal bytes -> merge
    a = g.add_node("ADD", [x, y])
    b = g.add_node("ADD", [y, x])   # commutative -> merges into a
    ea = g.add_node("EXP", [a])
    eb = g.add_node("EXP", [b])     # cascades
    s = g.add_node("SUB", [ea, eb])
    t = g.add_node("SUB", [eb, ea])  # becomes SUB(ea, ea) == s after the cascade
    d1 = g.add_node("DIV", [ea, x])
    d2 = g.add_node("DIV", [x, ea])  # DIV not commutative -> distinct
    u = g.add_node("MUL", [s, k1])
    w = g.add_node("MUL", [t, k2])   # -> MUL(s, k1) == u
    z = g.add_node("ADD", [u, w])
    q = g.add_node("ADD", [g.add_node("ADD", [z, x2]), g.add_node("ADD", [d1, d2])])
    c = compile_graph(g, [q])
    assert c.opt.rep == {k2: k1, b: a, eb: ea, t: s, w: u}
    assert c.g.nodes[z].preds == [u, u] and c.g.nodes[d2].preds == [x, ea]
    assert c.opt.report["cse_merged"] == 5


def test_c2_structure():
    """CSE merges 15->6, CF folds n1, n2, DCE drops kb, kc; 17 ops, 1 group."""
    g, outs = from_spec(configs.c2(rows=8, cols=16))
    c = compile_graph(g, outs)
    assert {k: c.opt.report[k] for k in ("cse_merged", "cf_folded", "dce_removed")} == {"cse_merged": 1, "cf_folded": 2, "dce_removed": 2}
    assert c.opt.rep == {23: 14} and c.opt.folded == [9, 10] and sorted(c.opt.dead) == [6, 7, 23]
    assert float(c.g.nodes[9].value) == 1.0 and c.g.nodes[10].value == np.float32(0.044715)
    assert len(c.groups) == 1 and len(c.groups[0].members) == 17
    assert sorted(c.groups[0].inputs) == [0, 1, 2, 3, 4, 5, 8, 9, 10]
    assert c.plan.size == [8 * 16 * 4]


# ---------------------------------------------------------------- Alg. 1
def test_find_best_block_examples():
    size = [4, 10]
    assert find_best_block({0, 1}, size, 6) == (1, False)          # S:281 smallest >= s
    size = [4]
    reus = {0}
    assert find_best_block(reus, size, 6) == (0, False) and size == [6] and not reus  # S:282 grow
    size = []
    assert find_best_block(set(), size, 8) == (0, True) and size == [8]             # S:283 new


@pytest.mark.parametrize("flags,blocks", [(FLAG_NO_FUSION, [4096]), (0, [4096]),
                                          (FLAG_INCREMENTAL, [4096, 4096]),
                                          (FLAG_INCREMENTAL | FLAG_NO_FUSION, [4096] * 3)])
def test_plan_traces_fig1(flags, blocks):
    g, outs = _fig1()
    g, outs = from_spec(configs.c1(1024))
    c = compile_graph(g, outs, flags)
    assert c.plan.size == blocks
    if flags == FLAG_NO_FUSION:
        assert c.plan.block == {2: 0, 4: 0, 5: 0}  # x4 slides into x2, x5 into x4
        assert c.unshared_bytes == 3 * 4096
    if flags == 0:
        assert [G.members for G in c.groups] == [[2, 4, 5]]
    if flags == FLAG_INCREMENTAL:
        assert [G.members for G in c.groups] == [[2], [4, 5]]
    assert validate_plan(c) == []


def _fig3():
    g = Graph()
    v0 = g.add_leaf("VAR", [1024])
    n1 = g.add_node("SIN", [v0])
    n2 = g.add_node("COS", [n1])
    v3 = g.add_leaf("VAR", [1024])
    n4 = g.add_node("MUL", [n2, v3])
    n5 = g.add_node("ADD", [n1, n4])
    return g, [n5]


def test_plan_trace_fig3():
    g, outs = _fig3()
    # edge list of hardpebbling: 0->1, 1->5, 1->2, 2->4, 3->4, 4->5
    assert sorted((p, n.id) for n in g.nodes for p in n.preds) == [(0, 1), (1, 2), (1, 5), (2, 4), (3, 4), (4, 5)]
    c = compile_graph(g, outs, FLAG_NO_FUSION)
    assert c.gamma == [0, 1, 2, 3, 4, 5]
    # 1->B0; 2->B1 (1 still needed by 5); 4 slides into B1; 5 takes B0 (tie -> lowest id)
    assert c.plan.block == {1: 0, 2: 1, 4: 1, 5: 0} and len(c.plan.size) == 2
    c = compile_graph(g, outs, 0)
    assert [G.members for G in c.groups] == [[1, 2, 4, 5]]


def test_chain_and_matmul_traces():
    g = Graph()
    x = g.add_leaf("VAR", [64])
    v = x
    for k in range(10):
        v = g.add_node(["NEG", "EXP", "SIN", "COS", "TANH"][k % 5], [v])
    c = compile_graph(g, [v], FLAG_NO_FUSION)
    assert len(c.plan.size) == 1
    g = Graph()
    a = g.add_leaf("VAR", [8, 8])
    b = g.add_leaf("VAR", [8, 8])
    ea = g.add_node("EXP", [a])
    eb = g.add_node("EXP", [b])
    m = g.add_node("DOT", [ea, eb], {"ta": 0, "tb": 0})
    c = compile_graph(g, [m], FLAG_NO_FUSION)
    assert c.plan.block[m] not in (c.plan.block[ea], c.plan.block[eb])
    assert len(c.plan.size) == 3


def test_broadcast_input_not_overwritten_in_place():
    """R13: a dying broadcast input of an elementwise group is released after allocation."""
    g = Graph()
    x = g.add_leaf("VAR", [1, 64])
    y = g.add_leaf("VAR", [32, 64])
    big = g.add_node("EXP", [y])              # 8 KiB block B0
    red = g.add_node("SUM", [big], {"a0": 0, "a1": 1})  # [1,64] -> B1; big dies -> B0 reusable
    r2 = g.add_node("ADD", [red, x])          # [1,64] elementwise: takes B0 (best fit), red stays in B1
    out = g.add_node("MUL", [r2, y])          # [32,64] broadcast read of r2 (dies here)
    c = compile_graph(g, [out], FLAG_NO_FUSION)
    assert c.plan.block[out] != c.plan.block[r2]
    assert validate_plan(c) == []


def test_validator_catches_bad_plans():
    g, outs = _fig3()
    c = compile_graph(g, outs, FLAG_NO_FUSION)
    bad = dict(c.plan.block)
    bad[2] = 0  # 2 shares B0 with 1 while 1 is live until 5
    assert any("overlap" in e for e in validate_plan(c, block=bad))
    assert any("undersized" in e for e in validate_plan(c, size=[8, 4096]))
    g = Graph()
    a = g.add_leaf("VAR", [8, 8])
    ea = g.add_node("EXP", [a])
    m = g.add_node("DOT", [ea, ea], {"ta": 0, "tb": 0})
    c = compile_graph(g, [m], FLAG_NO_FUSION)
    assert any("overlap" in e for e in validate_plan(c, block={ea: 0, m: 0}, size=[256]))


def test_plan_scales_n_log_b():
    """10k-node plan well under a few seconds even in the slow oracle (S:308 sanity)."""
    import time
    g = Graph()
    x = g.add_leaf("VAR", [16])
    v = x
    for k in range(10000):
        v = g.add_node("NEG" if k % 2 else "EXP", [v])
    t = time.time()
    c = compile_graph(g, [v], FLAG_NO_FUSION, compute_values=False)
    assert time.time() - t < 20 and len(c.plan.size) == 1


# ---------------------------------------------------------------- closed forms
def _run1(op, ins, attrs=None):
    g = Graph()
    ids = [g.add_leaf("VAR", np.shape(a)) for a in ins]
    o = g.add_node(op, ids, attrs or {})
    v = evaluate(g, leaf_values(g, dict(zip(ids, ins))))
    return v[o]


def test_reduction_closed_forms():
    n = 4000
    x = np.arange(n, dtype=np.float32).reshape(40, 100)
    assert _run1("SUM", [x], {"a0": 0, "a1": 2})[0, 0] == n * (n - 1) / 2
    assert np.array_equal(_run1("SUM", [x], {"a0": 1, "a1": 2})[:, 0],
                          [100 * (100 * r) + 4950 for r in range(40)])
    assert np.array_equal(_run1("MAX", [x], {"a0": 0, "a1": 1})[0], x[-1])


def test_dot_brute_force_exact():
    rng = np.random.default_rng(0)
    A = rng.integers(-4, 5, (5, 7)).astype(np.float32)
    B = rng.integers(-4, 5, (7, 3)).astype(np.float32)
    C = np.zeros((5, 3))
    for i in range(5):
        for j in range(3):
            for k in range(7):
                C[i, j] += float(A[i, k]) * float(B[k, j])
    assert np.array_equal(_run1("DOT", [A, B], {"ta": 0, "tb": 0}), C)
    assert np.array_equal(_run1("DOT", [A.T.copy(), B.T.copy()], {"ta": 1, "tb": 1}), C)


def _conv_loops(x, w, sh, sw, pad):
    n, h, wd, ci = x.shape
    KH, KW, _, co = w.shape
    ho, pt = ops.conv_out(h, KH, sh, pad)
    wo, pl = ops.conv_out(wd, KW, sw, pad)
    y = np.zeros((n, ho, wo, co))
    for b in range(n):
        for i in range(ho):
            for j in range(wo):
                for kh in range(KH):
                    for kw in range(KW):
                        hi, wi = i * sh + kh - pt, j * sw + kw - pl
                        if 0 <= hi < h and 0 <= wi < wd:
                            for c in range(ci):
                                for o in range(co):
                                    y[b, i, j, o] += float(x[b, hi, wi, c]) * float(w[kh, kw, c, o])
    return y


@pytest.mark.parametrize("sh,pad", [(1, 0), (1, 1), (2, 0), (2, 1)])
def test_conv_brute_force_and_adjoint(sh, pad):
    rng = np.random.default_rng(sh * 10 + pad)
    x = rng.integers(-3, 4, (2, 7, 6, 3)).astype(np.float32)
    w = rng.integers(-3, 4, (3, 2, 3, 4)).astype(np.float32)
    a = {"sh": sh, "sw": sh, "pad": pad}
    y = _run1("CONV2D", [x, w], a)
    assert np.array_equal(y, _conv_loops(x, w, sh, sh, pad))  # integers: exact
    # adjoint identities <conv(x,w), dy> = <x, bwd_in(dy,w)> = <w, bwd_k(x,dy)>
    xf = rng.standard_normal(x.shape)
    wf = rng.standard_normal(w.shape)
    dy = rng.standard_normal(y.shape)
    yv = ops.conv2d_f64(xf, wf, sh, sh, pad)
    dx = ops.conv2d_bwd_input_f64(dy, wf, 7, 6, sh, sh, pad)
    dw = ops.conv2d_bwd_kernel_f64(xf, dy, 3, 2, sh, sh, pad)
    lhs = np.sum(yv * dy)
    assert abs(lhs - np.sum(xf * dx)) < 1e-10 * max(1, abs(lhs))
    assert abs(lhs - np.sum(wf * dw)) < 1e-10 * max(1, abs(lhs))


def test_pool_brute_force():
    rng = np.random.default_rng(3)
    x = rng.integers(0, 3, (2, 5, 6, 2)).astype(np.float32)  # many ties
    for k, s, pad in [(2, 2, 0), (3, 2, 0), (3, 1, 1), (3, 2, 1)]:
        a = {"kh": k, "kw": k, "sh": s, "sw": s, "pad": pad}
        ho, pt = ops.conv_out(5, k, s, pad)
        wo, pl = ops.conv_out(6, k, s, pad)
        mx = np.full((2, ho, wo, 2), -np.inf)
        av = np.zeros((2, ho, wo, 2))
        dx = np.zeros(x.shape)
        dy = rng.integers(1, 5, (2, ho, wo, 2)).astype(np.float32)
        for b in range(2):
            for i in range(ho):
                for j in range(wo):
                    for c in range(2):
                        cells = [(i * s + kh - pt, j * s + kw - pl) for kh in range(k) for kw in range(k)]
                        cells = [(h, w) for h, w in cells if 0 <= h < 5 and 0 <= w < 6]
                        vals = [x[b, h, w, c] for h, w in cells]
                        mx[b, i, j, c] = max(vals)
                        av[b, i, j, c] = sum(vals) / len(vals)
                        first = cells[vals.index(max(vals))]
                        dx[b, first[0], first[1], c] += dy[b, i, j, c]
        assert np.array_equal(_run1("MAXPOOL2D", [x], a), mx)
        assert np.allclose(_run1("AVGPOOL2D", [x], a), av, rtol=1e-7)
        assert np.array_equal(_run1("MAXPOOL2D_BWD", [x, dy], a), dx)


def test_elementwise_identities():
    x = np.linspace(0.1, 3.0, 97, dtype=np.float32)
    assert np.array_equal(_run1("RELU", [x - 1.5]), np.maximum(x - 1.5, 0))
    assert np.array_equal(_run1("RELU_GRAD", [x - 1.5, x]), np.where(x - 1.5 > 0, x, 0))
    # + - * / sqrt: f64-then-round == correctly rounded fp32 == numpy fp32 IEEE
    y = x[::-1].copy()
    for op, f in [("ADD", np.add), ("SUB", np.subtract), ("MUL", np.multiply), ("DIV", np.divide)]:
        assert np.array_equal(_run1(op, [x, y]), f(x, y))
    assert np.array_equal(_run1("SQRT", [x]), np.sqrt(x))
    e = _run1("EXP", [_run1("LOG", [x])])
    assert np.max(np.abs(e - x) / x) < 2e-7
    t = _run1("TANH", [x])
    assert np.array_equal(_run1("TANH", [-x]), -t)
    assert np.allclose(_run1("FMA", [x, y, x]), x.astype(np.float64) * y + x, rtol=6e-8)


def test_pow_closed_forms():
    """POW (S:133 binary op list; numpy power semantics, DESIGN §3 c1) pinned by
    what the mathematics fixes: x^2 = x*x and x^0.5 = sqrt(x) (both correctly
    rounded in fp32 — the f64 product of two fp32 values is exact), x^1 = x,
    x^0 = 1 (0^0 = 1 as in C99 pow), 2^3 = 8 and 3^2 = 9 (operand order),
    x^-1 = 1/x, integer powers by repeated products, a negative base with a
    non-integer exponent is NaN, 0^-1 = +inf."""
    x = np.linspace(0.05, 7.0, 211, dtype=np.float32)
    two = np.full_like(x, 2.0)
    assert np.array_equal(_run1("POW", [x, two]), x * x)
    assert np.array_equal(_run1("POW", [-x, two]), x * x)
    assert np.array_equal(_run1("POW", [x, np.full_like(x, 0.5)]), np.sqrt(x))
    assert np.array_equal(_run1("POW", [x, np.ones_like(x)]), x)
    assert np.all(_run1("POW", [np.concatenate([x, [0.0, -3.0]]).astype(np.float32),
                                np.zeros(213, np.float32)]) == 1.0)
    assert _run1("POW", [np.float32([2.0]), np.float32([3.0])])[0] == 8.0
    assert _run1("POW", [np.float32([3.0]), np.float32([2.0])])[0] == 9.0
    assert np.array_equal(_run1("POW", [x, -np.ones_like(x)]), np.float32(1) / x)
    # x^3 = x*x*x to within the one extra rounding of the fp32 product chain
    cube = (x.astype(np.float64) ** 2) * x.astype(np.float64)
    assert np.max(np.abs(_run1("POW", [x, np.full_like(x, 3.0)]) - cube) / cube) < 6e-8
    assert np.all(np.isnan(_run1("POW", [np.float32([-2.0, -0.5]), np.float32([0.5, 1.5])])))
    assert _run1("POW", [np.float32([0.0]), np.float32([-1.0])])[0] == np.inf
    # broadcasting: a scalar exponent against a vector
    assert np.array_equal(_run1("POW", [x, np.float32(2.0)]), x * x)


def test_sign_and_selection_ops():
    """ABS / NEG / MAX2 / MIN2 / COS pinned by identities, not by re-typing them:
    |x| = max(x, -x); NEG is an involution that flips the sign bit (NEG(0) = -0);
    max(a, b) + min(a, b) = a + b and max(a, b) >= both operands (exact in fp32);
    NaN propagates through MAX2 / MIN2 (numpy maximum / minimum); cos 0 = 1,
    cos pi = -1, cos^2 + sin^2 = 1 and cos x = sin(pi/2 - x) to rounding."""
    rng = np.random.default_rng(7)
    a = rng.standard_normal(300).astype(np.float32)
    b = rng.standard_normal(300).astype(np.float32)
    ab = _run1("ABS", [a])
    assert np.array_equal(ab, np.where(a < 0, -a, a)) and np.all(np.signbit(ab) == False)  # noqa: E712
    assert np.signbit(_run1("ABS", [np.float32([-0.0])]))[0] == False  # noqa: E712
    n = _run1("NEG", [a])
    assert np.array_equal(_run1("NEG", [n]), a) and np.all(n + a == 0)
    assert np.signbit(_run1("NEG", [np.float32([0.0])]))[0]
    mx, mn = _run1("MAX2", [a, b]), _run1("MIN2", [a, b])
    assert np.array_equal(mx + mn, a + b)
    assert np.all(mx >= a) and np.all(mx >= b) and np.all(mn <= a) and np.all(mn <= b)
    assert np.all((mx == a) | (mx == b)) and np.all((mn == a) | (mn == b))
    nan = np.float32([np.nan, 1.0])
    assert np.isnan(_run1("MAX2", [nan, np.float32([5.0, 5.0])])[0])
    assert np.isnan(_run1("MIN2", [np.float32([5.0, 5.0]), nan])[0])
    c = _run1("COS", [np.float32([0.0, np.pi])])
    assert c[0] == 1.0 and c[1] == -1.0
    s_ = _run1("SIN", [a]).astype(np.float64)
    c_ = _run1("COS", [a]).astype(np.float64)
    assert np.max(np.abs(s_ * s_ + c_ * c_ - 1)) < 2e-7
    shifted = (np.float64(np.pi / 2) - a.astype(np.float64))
    assert np.max(np.abs(c_ - np.sin(shifted))) < 1e-7


def test_concat_and_reshape_values():
    """CONCAT places its operands side by side along the axis (slicing the result
    returns them); RESHAPE keeps row-major element order (the flat index of
    [i, j] in a [R, C] view is i*C + j), so reshaping arange gives arange."""
    a = np.arange(24, dtype=np.float32).reshape(2, 3, 4)
    b = -np.arange(16, dtype=np.float32).reshape(2, 2, 4)
    cat = _run1("CONCAT", [a, b], {"axis": 1})
    assert cat.shape == (2, 5, 4)
    assert np.array_equal(cat[:, :3], a) and np.array_equal(cat[:, 3:], b)
    c = _run1("CONCAT", [a, a[:, :, :1]], {"axis": 2})
    assert np.array_equal(c[..., 4], a[..., 0]) and np.array_equal(c[..., :4], a)
    r = _run1("RESHAPE", [a], {"dims": [4, 6]})
    for i in range(4):
        for j in range(6):
            assert r[i, j] == i * 6 + j


def test_softmax_rows_sum_to_one():
    g = Graph()
    L = g.add_leaf("VAR", [6, 10])
    M = g.add_node("MAX", [L], {"a0": 1, "a1": 2})
    E = g.add_node("EXP", [g.add_node("SUB", [L, M])])
    P = g.add_node("DIV", [E, g.add_node("SUM", [E], {"a0": 1, "a1": 2})])
    v = evaluate(g, leaf_values(g, {L: np.random.default_rng(1).standard_normal((6, 10)) * 5}))
    assert np.allclose(v[P].astype(np.float64).sum(axis=1), 1.0, atol=1e-6)


# ---------------------------------------------------------------- dumps
def test_dump_determinism_and_format():
    spec = configs.c2(rows=8, cols=16)
    g, outs = from_spec(spec)
    c1 = compile_graph(g, outs)
    g2, _ = from_spec(spec)
    c2 = compile_graph(g2, outs)
    assert graph_json(c1.opt) == graph_json(c2.opt) and plan_json(c1) == plan_json(c2)
    s = plan_json(c1)
    assert " " not in s and s.startswith('{"block":[[')
