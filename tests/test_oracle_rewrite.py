"""f1 rewrites (oracle/rewrite.py) pinned by hand-built graphs, the
paper's patterns, a closed form, fixpoint and semantics preservation."""
import numpy as np
import pytest

from oracle.dump import compile_graph
from oracle.eager import ancestors, evaluate, leaf_values
from oracle.graph import Graph, from_spec
from oracle.rewrite import RW_ADAGRAD, RW_ALL, RW_FMA, RW_IDENTITY
from tests.randgraph import random_spec
from workloads import configs


def _g():
    g = Graph()
    x = g.add_leaf("VAR", (4, 8), data={"kind": "uniform", "tag": "x", "lo": -1, "hi": 1})
    y = g.add_leaf("VAR", (4, 8), data={"kind": "uniform", "tag": "y", "lo": -1, "hi": 1})
    z = g.add_leaf("VAR", (4, 8), data={"kind": "uniform", "tag": "z", "lo": -1, "hi": 1})
    return g, x, y, z


def _live_ops(c):
    return sum(1 for n in c.opt.g.nodes if n.id not in c.opt.dead and n.op not in ("VAR", "CONST"))


def _eval_opt(c, raw_leaves):
    vals = dict(raw_leaves)
    for n in c.opt.g.nodes:
        if n.op == "CONST" and n.id not in c.opt.dead:
            vals[n.id] = c.opt.g.const_value(n.id)
    need = ancestors(c.opt.g, c.outputs)
    return evaluate(c.opt.g, vals, need)


def test_fma_pattern_drops_one_node():
    g, x, y, z = _g()
    m = g.add_node("MUL", [x, y])
    a = g.add_node("ADD", [m, z])
    c0 = compile_graph(g, [a], 0, rewrites=0)
    c = compile_graph(g, [a], 0, rewrites=RW_FMA)
    assert _live_ops(c0) - _live_ops(c) == 1
    assert c.opt.g.nodes[a].op == "FMA" and c.opt.g.nodes[a].preds == [x, y, z] and m in c.opt.dead
    assert c.opt.report["rw_fma"] == 1
    leaves = leaf_values(g)
    want = (leaves[x].astype(np.float64) * leaves[y] + leaves[z]).astype(np.float32)  # one rounding
    assert np.array_equal(_eval_opt(c, leaves)[a], want)


def test_fma_needs_single_consumer_and_goes_left_first():
    g, x, y, z = _g()
    m = g.add_node("MUL", [x, y])
    a = g.add_node("ADD", [m, z])
    b = g.add_node("NEG", [m])
    c = compile_graph(g, [a, b], 0, rewrites=RW_FMA)
    assert c.opt.report["rw_fma"] == 0
    g, x, y, z = _g()
    m1 = g.add_node("MUL", [x, y])
    m2 = g.add_node("MUL", [y, z])
    a = g.add_node("ADD", [m1, m2])
    c = compile_graph(g, [a], 0, rewrites=RW_FMA)
    assert c.opt.g.nodes[a].op == "FMA" and c.opt.g.nodes[a].preds == [x, y, m2]


def _adagrad_graph(share_sqrt=False):
    g = Graph()
    gr = g.add_leaf("VAR", (6,), data={"kind": "uniform", "tag": "g", "lo": -1, "hi": 1})
    s = g.add_leaf("VAR", (6,), data={"kind": "uniform", "tag": "s", "lo": 0.5, "hi": 2})
    lr = g.add_leaf("CONST", (), data={"kind": "literal", "values": [0.1]})
    eps = g.add_leaf("CONST", (), data={"kind": "literal", "values": [1e-8]})
    num = g.add_node("MUL", [lr, gr])
    q = g.add_node("SQRT", [s])
    den = g.add_node("ADD", [q, eps])
    d = g.add_node("DIV", [num, den])
    outs = [d] + ([g.add_node("NEG", [q])] if share_sqrt else [])
    return g, outs, (gr, s, lr, eps, num, q, den, d)


def test_adagrad_pattern_and_closed_form():
    g, outs, (gr, s, lr, eps, num, q, den, d) = _adagrad_graph()
    c = compile_graph(g, outs, 0, rewrites=RW_ADAGRAD)
    n = c.opt.g.nodes[d]
    assert n.op == "FUSED_ADAGRAD" and n.preds == [gr, s, lr, eps]
    assert {num, q, den} <= c.opt.dead and c.opt.report["rw_adagrad"] == 1
    # FusedAdagrad(lr=0.1, eps=1e-8)(g=1, s=4) = 0.1*1/(2+1e-8) ~ 0.05
    val = _eval_opt(c, {gr: np.ones(6, np.float32), s: np.full(6, 4, np.float32)})[d]
    assert np.allclose(val, 0.05, rtol=1e-6)
    g, outs, _ = _adagrad_graph(share_sqrt=True)
    assert compile_graph(g, outs, 0, rewrites=RW_ADAGRAD).opt.report["rw_adagrad"] == 0


def test_identities():
    g, x, y, z = _g()
    one = g.add_leaf("CONST", (4, 8), data={"kind": "full", "value": 1.0})
    zero = g.add_leaf("CONST", (), data={"kind": "literal", "values": [0.0]})
    big0 = g.add_leaf("CONST", (3, 4, 8), data={"kind": "full", "value": 0.0})
    a = g.add_node("MUL", [x, one])          # -> x
    b = g.add_node("ADD", [a, zero])         # -> x
    k = g.add_node("ADD", [y, big0])         # broadcasting changes the shape: kept
    m = g.add_node("MUL", [z, zero])         # -> Const zeros
    t = g.add_node("SUB", [b, m])            # x - 0 -> x ... after the zero rewrite
    out = g.add_node("NEG", [t])
    c = compile_graph(g, [out, k], 0, rewrites=RW_IDENTITY)
    assert c.opt.g.nodes[out].preds == [x]
    assert c.opt.rep[a] == x and c.opt.rep[b] == x and c.opt.rep[t] == x
    assert c.opt.g.nodes[k].op == "ADD" and c.opt.g.nodes[m].op == "CONST"
    assert c.opt.report["rw_identity"] == 3 and c.opt.report["rw_zeroed"] == 1
    leaves = leaf_values(g)
    assert np.array_equal(_eval_opt(c, leaves)[out], -leaves[x])


def test_fig1_unchanged_and_fixpoint():
    spec = configs.c1(16)
    og, oo = from_spec(spec)
    c = compile_graph(og, oo, 0, rewrites=RW_ALL)
    assert sum(c.opt.rewrites[k] != [] for k in c.opt.rewrites) == 0
    g, x, y, z = _g()
    m = g.add_node("MUL", [x, y])
    a = g.add_node("ADD", [m, z])
    c1 = compile_graph(g, [a], 0, rewrites=RW_ALL)
    c2 = compile_graph(c1.opt.g, [a], 0, rewrites=RW_ALL)
    assert all(v == [] for v in c2.opt.rewrites.values())


@pytest.mark.parametrize("seed", range(60))
def test_rewrites_preserve_semantics(seed):
    spec = random_spec(seed, allow_updates=False, simple_values=True)
    og, oo = from_spec(spec)
    c = compile_graph(og, oo, 0, rewrites=RW_ALL)
    raw = evaluate(og, leaf_values(og))
    got = _eval_opt(c, leaf_values(og))
    for o0, o in zip(oo, c.outputs):
        want, have = raw[o0].astype(np.float64), got[o].astype(np.float64)
        fin = np.isfinite(want)
        assert np.array_equal(fin, np.isfinite(have))
        if fin.any():
            m = np.max(np.abs(want[fin]))
            assert m == 0 or np.max(np.abs(have[fin] - want[fin])) / m <= 1e-5
    assert _live_ops(c) <= sum(1 for n in og.nodes if n.op not in ("VAR", "CONST"))


def test_c3_adagrad_variant():
    spec = configs.c3(batch=64, widths=(784, 64, 32, 10), optimizer="adagrad")
    og, oo = from_spec(spec)
    c = compile_graph(og, oo, 0, rewrites=RW_ALL)
    assert c.opt.report["rw_adagrad"] == 6 and c.opt.report["rw_fma"] >= 6
