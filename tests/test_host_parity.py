"""Host-compiler parity (CPU): the C++ library in host-only mode vs the oracle.

The structural products — rewritten graph (CSE/CF/DCE), gamma, fusion groups,
Algorithm 1 memory plan — must match the oracle BYTE-FOR-BYTE (north star:
"Memory plans, CSE and fusion groupings must match bit-exactly").  Both sides
implement DESIGN.md's readings independently and share no code.
Also: the library exports every symbol include/*.h declares, reports the
documented error codes, and every generated kernel compiles for sm_100a with
NVRTC (no GPU needed).
"""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

from oracle.dump import compile_graph, graph_json, plan_json
from oracle.graph import from_spec
from paper_1812_03770_b200 import cg
from tests.randgraph import random_spec
from workloads import configs
from workloads.gen import materialise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODES = [0, cg.PLAN_INCREMENTAL, cg.PLAN_NO_FUSION, cg.PLAN_INCREMENTAL | cg.PLAN_NO_FUSION]


def _const_data(rec):
    return materialise(rec["data"], rec["shape"]) if rec["op"] == "CONST" else None


def host_graph(spec, flags, optimise=True, rewrites=0):
    g, outs = cg.build_from_spec(spec, device=-1, data_fn=_const_data)
    if rewrites:
        g.set_rewrites(rewrites)
    rep = g.optimise(outs) if optimise else None
    info = g.plan_memory(outs, flags)
    return g, outs, rep, info


def check_parity(spec, flags, rewrites=0):
    g, outs, rep, info = host_graph(spec, flags, rewrites=rewrites)
    og, oo = from_spec(spec)
    c = compile_graph(og, oo, flags, compute_values=False, rewrites=rewrites)
    assert rep == c.opt.report
    assert g.dump_json(cg.DUMP_GRAPH) == graph_json(c.opt)
    assert g.dump_json(cg.DUMP_PLAN) == plan_json(c)
    assert info["n_groups"] == len(c.groups) and info["n_blocks"] == len(c.plan.size)
    assert info["pool_bytes"] == c.plan.pool_bytes and info["unshared_bytes"] == c.unshared_bytes
    return g


def test_abi_symbols_exported():
    L = ctypes.CDLL(cg.LIB_PATH)
    declared = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        # function declarations: a line starting with a return type, then the name and "("
        declared |= set(re.findall(r"^[A-Za-z_][\w \*]*?\b(cgx?_[a-z0-9_]+)\s*\(", txt, re.M))
    assert {"cg_create", "cg_add_node", "cg_add_update", "cg_optimise", "cg_plan_memory", "cg_assign",
            "cg_eval", "cg_destroy"} <= declared
    for name in sorted(declared):
        assert hasattr(L, name), name


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
@pytest.mark.parametrize("flags", MODES)
def test_config_parity(name, flags):
    spec = {"C1": lambda: configs.c1(), "C2": lambda: configs.c2(),
            "C3": lambda: configs.c3(), "C4": lambda: configs.c4()}[name]()
    check_parity(spec, flags)


def test_c5_parity_and_memory():
    """InceptionV3-shaped graph at batch 256: plan exact, peak << unshared (P:379 motivation)."""
    spec = configs.c5()
    g = check_parity(spec, 0)
    info = g.plan_memory.__self__ if False else None  # noqa: F841
    og, oo = from_spec(spec)
    c = compile_graph(og, oo, 0, compute_values=False)
    assert c.opt.report["cf_folded"] == 94 and c.opt.report["dce_removed"] >= 94
    assert c.plan.pool_bytes < c.unshared_bytes / 10


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C3adagrad"])
def test_rewrite_parity_configs(name):
    """f1 rewrites: the C++ host compiler and the oracle rewrite the
    same nodes, byte for byte (graph and plan dumps, rewrite counts)."""
    spec = configs.c3(optimizer="adagrad") if name == "C3adagrad" else configs.CONFIGS[name]()
    g = check_parity(spec, 0, rewrites=cg.RW_ALL)
    if name == "C3adagrad":
        assert '"adagrad":[' in g.dump_json(cg.DUMP_GRAPH)


@pytest.mark.parametrize("flags", [0, cg.PLAN_NO_FUSION])
def test_rewrite_parity_random(flags):
    for seed in range(200):
        check_parity(random_spec(seed, rewrite_bait=True), flags, rewrites=cg.RW_ALL)


@pytest.mark.parametrize("flags", MODES)
def test_random_dag_parity(flags):
    for seed in range(250):
        check_parity(random_spec(seed), flags)


def test_no_optimise_parity():
    for seed in range(100):
        spec = random_spec(1000 + seed)
        g, outs, _, _ = host_graph(spec, 0, optimise=False)
        og, oo = from_spec(spec)
        c = compile_graph(og, oo, 0, do_optimise=False)
        assert g.dump_json(cg.DUMP_PLAN) == plan_json(c)


def test_abi_errors():
    g = cg.Graph(-1)
    x = g.var([2, 3])
    y = g.var([3, 2])
    with pytest.raises(cg.CGError) as e:
        g.add_node("ADD", [x])
    assert e.value.code == "CG_E_ARITY"
    with pytest.raises(cg.CGError) as e:
        g.add_node("NEG", [9])
    assert e.value.code == "CG_E_BAD_NODE"
    with pytest.raises(cg.CGError) as e:
        g.add_node("ADD", [x, y])
    assert e.value.code == "CG_E_SHAPE"
    m = g.add_node("NEG", [x])
    with pytest.raises(cg.CGError) as e:
        g.add_update(x, m)
    assert e.value.code == "CG_E_NOT_VAR"
    with pytest.raises(cg.CGError) as e:
        g.add_update(m, y)
    assert e.value.code == "CG_E_UPDATE_SHAPE"
    g.add_update(m, x)
    with pytest.raises(cg.CGError) as e:
        g.add_update(m, x)
    assert e.value.code == "CG_E_DUP_UPDATE"
    g.plan_memory([m])
    with pytest.raises(cg.CGError) as e:
        g.add_node("NEG", [m])
    assert e.value.code == "CG_E_STATE"
    with pytest.raises(cg.CGError) as e:
        g.eval([m])
    assert e.value.code == "CG_E_NO_DEVICE"


def _codegen_check(g, sms=148):
    L = cg.lib()
    f = L.cgx_codegen_check
    f.restype = ctypes.c_int64
    f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    buf = ctypes.create_string_buffer(1 << 20)
    r = f(g.h, sms, buf, len(buf))
    assert r >= 0, buf.value.decode()[:6000]
    return r


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_generated_kernels_compile(name):
    spec = {"C1": lambda: configs.c1(), "C2": lambda: configs.c2(),
            "C3": lambda: configs.c3(), "C4": lambda: configs.c4()}[name]()
    for flags in (0, cg.PLAN_NO_FUSION):
        g, _, _, _ = host_graph(spec, flags)
        assert _codegen_check(g) >= 1


def test_generated_kernels_compile_random():
    n = 0
    for seed in range(0, 60):
        g, _, _, _ = host_graph(random_spec(seed), 0)
        n += _codegen_check(g)
    assert n > 60


def _rowrun_check(g, sms=148):
    L = cg.lib()
    f = L.cgx_rowrun_check
    f.restype = ctypes.c_int64
    f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    buf = ctypes.create_string_buffer(1 << 20)
    r = f(g.h, sms, buf, len(buf))
    assert r >= 0, buf.value.decode()[:6000]
    return r, buf.value.decode()


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_row_runs_generate_and_compile(name):
    """f2 reduce -> broadcast fusion: the softmax(-xent) groups of C3 / C4 / C5
    (MAX, SUB, EXP, SUM, LOG / DIV over [B, classes]) form row runs whose single
    kernel compiles (NVRTC, sm_100a)."""
    spec = {"C3": lambda: configs.c3(), "C4": lambda: configs.c4(), "C5": lambda: configs.c5(batch=2)}[name]()
    g, _, _, _ = host_graph(spec, 0)
    n, log = _rowrun_check(g)
    assert n >= 1, log
    runs = [tuple(int(x) for x in ln.split(":")[0].split("-")) for ln in log.split()]
    assert max(b - a + 1 for a, b in runs) >= 3, log  # MAX -> SUB/EXP -> SUM at least


def test_row_runs_compile_random():
    n = 0
    for seed in range(0, 40):
        g, _, _, _ = host_graph(random_spec(seed), 0)
        n += _rowrun_check(g)[0]
    assert n >= 0


# ---- R14 zero-copy CONCAT (f2; sub-block views, offset != 0 extension of P:303-310)
def _concat_spec(nested=False, twice=False, keep_a=False, reshape_b=False):
    from workloads.configs import Spec
    s = Spec("concat")
    x = s.var("x", [2, 3, 4], {"kind": "uniform", "tag": "x", "lo": -1.0, "hi": 1.0})
    y = s.var("y", [2, 3, 2], {"kind": "uniform", "tag": "y", "lo": -1.0, "hi": 1.0})
    a = s.op("RELU", x)
    b = s.op("RESHAPE", s.op("NEG", s.op("RESHAPE", y, dims=[2, 6])), dims=[2, 3, 2]) if reshape_b else s.op("NEG", y)
    c = s.op("CONCAT", a, b, a, axis=2) if twice else s.op("CONCAT", a, b, axis=2)
    if nested:
        d = s.op("EXP", y)
        c = s.op("CONCAT", c, d, axis=2)
    s.output(s.op("SIN", c))
    if keep_a:
        s.output(a)
    return s.to_dict(), (x, y, a, b, c)


def _plan(spec, flags=0):
    og, oo = from_spec(spec)
    return compile_graph(og, oo, flags, compute_values=False)


def test_concat_views_oracle_pins():
    """The view tuples are fixed by the concat layout: element (o, i) of input v
    is element o * inner(root) + offset + i of the root (axis 2 of [2,3,*])."""
    from oracle.validate import validate_plan
    spec, (x, y, a, b, c) = _concat_spec()
    cp = _plan(spec)
    assert cp.plan.views == {a: (c, 6, 6, 0, 4), b: (c, 6, 6, 4, 2)}
    assert cp.plan.block[a] == cp.plan.block[b] == cp.plan.block[c]
    assert validate_plan(cp) == []
    # the mapping reproduces numpy concatenation exactly
    rng = np.random.default_rng(0)
    va, vb = rng.standard_normal((2, 3, 4)), rng.standard_normal((2, 3, 2))
    root = np.zeros(2 * 3 * 6)
    for v, val in ((a, va), (b, vb)):
        _, outer, inner_root, off, inner = cp.plan.views[v]
        flat = val.reshape(outer, inner)
        for o in range(outer):
            root[o * inner_root + off: o * inner_root + off + inner] = flat[o]
    assert np.array_equal(root.reshape(2, 3, 6), np.concatenate([va, vb], axis=2))
    check_parity(spec, 0)
    check_parity(spec, cg.PLAN_NO_FUSION)


def test_concat_views_nested_and_refusals():
    from oracle.validate import validate_plan
    spec, (x, y, a, b, c) = _concat_spec(nested=True)
    cp = _plan(spec)
    inner_c, outer_c = [n["id"] for n in spec["nodes"] if n["op"] == "CONCAT"]
    assert c == outer_c
    d = [n["id"] for n in spec["nodes"] if n["op"] == "EXP"][0]
    # the inner concat is a view of the outer one; its inputs map to the same root
    assert cp.plan.views[inner_c] == (outer_c, 6, 8, 0, 6)
    assert cp.plan.views[a] == (outer_c, 6, 8, 0, 4) and cp.plan.views[b] == (outer_c, 6, 8, 4, 2)
    assert cp.plan.views[d] == (outer_c, 6, 8, 6, 2)
    assert validate_plan(cp) == []
    check_parity(spec, 0)
    # refusals: an input used twice, a kept input, a RESHAPE producer, incremental plans
    spec2, (_, _, a2, b2, _) = _concat_spec(twice=True)
    assert a2 not in _plan(spec2).plan.views and b2 in _plan(spec2).plan.views
    spec3, (_, _, a3, b3, _) = _concat_spec(keep_a=True)
    assert a3 not in _plan(spec3).plan.views and b3 in _plan(spec3).plan.views
    spec4, (_, _, a4, b4, _) = _concat_spec(reshape_b=True)
    assert b4 not in _plan(spec4).plan.views and a4 in _plan(spec4).plan.views
    assert _plan(spec, cg.PLAN_INCREMENTAL).plan.views == {}
    for sp in (spec2, spec3, spec4):
        check_parity(sp, 0)
    check_parity(spec, cg.PLAN_INCREMENTAL)
