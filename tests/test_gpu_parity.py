"""GPU parity: the CUDA path (through the C ABI) vs the oracle on the same seeded inputs.

Tolerances (north star): normwise max error <= 1e-5 for
elementwise / reduction graphs, <= 1e-3 for dot/conv training graphs after 10
iterations; bit-exact for IEEE-only chains (+ - * / sqrt round identically),
for integer-valued dot/conv/pool inputs, and for all structural integers
(eval counts, plans).
"""
import math

import numpy as np
import pytest

from oracle.dump import compile_graph
from oracle.eager import ancestors, apply_updates, evaluate, leaf_values
from oracle.graph import Graph as OGraph
from oracle.graph import from_spec
from oracle.incremental import IncrementalModel
from paper_1812_03770_b200 import cg
from tests.gpu_util import evaluate_pinned, gpu_graph, leaf_data, normwise, oracle_outputs, oracle_trajectory
from tests.randgraph import random_spec
from workloads import configs
from workloads.gen import materialise, retag

pytestmark = pytest.mark.gpu

MODES = [0, cg.PLAN_INCREMENTAL, cg.PLAN_NO_FUSION, cg.PLAN_INCREMENTAL | cg.PLAN_NO_FUSION]


# ---------------------------------------------------------------- C1 (Fig. 1)
@pytest.mark.parametrize("flags", MODES)
def test_c1_values_and_incremental(flags):
    spec = configs.c1(1024)
    g, outs, _, info = gpu_graph(spec, flags)
    g.eval(outs)
    ref, og, _ = oracle_outputs(spec)
    assert normwise(g.read(5), ref[5]) <= 1e-5
    assert [g.eval_count(v) for v in (2, 4, 5)] == [1, 1, 1]
    # change x3 only and re-evaluate
    x3 = materialise(spec["meta"]["reassign"]["x3"], [1024])
    g.assign(3, x3)
    g.eval(outs)
    ref2, _, _ = oracle_outputs(spec, {3: x3})
    assert normwise(g.read(5), ref2[5]) <= 1e-5
    assert g.eval_count(4) == 2 and g.eval_count(5) == 2
    if flags & cg.PLAN_INCREMENTAL:
        assert g.eval_count(2) == 1  # "no need to re-evaluate x2"
    # the oracle's c9 model predicts every count exactly
    c = compile_graph(og, [5], flags)
    m = IncrementalModel(c)
    m.eval([5])
    m.assign(3)
    m.eval([5])
    assert [g.eval_count(v) for v in (2, 4, 5)] == [m.count[v] for v in (2, 4, 5)]
    # x1 = 2 -> exactly zero
    g.assign(1, np.full(1024, 2.0, np.float32))
    g.eval(outs)
    assert np.all(g.read(5) == 0)


def test_c1_ieee_prefix_bit_exact():
    """x2 = 2 - x1 and x4 = x2 * x3 are IEEE ops: GPU == oracle bit for bit."""
    spec = configs.c1(4096)
    spec["outputs"] = [4, 5]
    g, outs, _, _ = gpu_graph(spec, 0)
    g.eval(outs)
    ref, _, _ = oracle_outputs(spec)
    assert np.array_equal(g.read(4), ref[4])
    assert normwise(g.read(5), ref[5]) <= 1e-5


def test_counter_three_rounds():
    g = cg.Graph(0)
    c = g.var([1])
    one = g.const(np.array(1.0, np.float32))
    c1 = g.add_node("ADD", [c, one])
    g.add_update(c1, c)
    g.plan_memory([c1])
    vals = []
    for _ in range(3):
        g.eval([c1])
        vals.append(float(g.read(c1)[0]))
    assert vals == [1.0, 2.0, 3.0] and float(g.read(c)[0]) == 3.0


# ---------------------------------------------------------------- C2 chain
@pytest.mark.parametrize("rows,cols", [(1000, 1024), (77, 256), (33, 20), (5, 4)])
def test_c2_small(rows, cols):
    spec = configs.c2(rows, cols)
    g, outs, rep, info = gpu_graph(spec, 0)
    assert {k: rep[k] for k in ("cse_merged", "cf_folded", "dce_removed")} == {"cse_merged": 1, "cf_folded": 2, "dce_removed": 2}
    assert info["n_groups"] == 1 and info["n_blocks"] == 1
    g.eval(outs)
    ref, _, _ = oracle_outputs(spec)
    assert normwise(g.read(outs[0]), ref[outs[0]]) <= 1e-5


def test_c2_full_size_sampled_rows():
    """BASELINE's full size [2^18, 1024] in the bench's launch configuration; the
    oracle recomputes 512 sampled rows (elementwise: row r depends on row r only)."""
    import torch
    spec = configs.c2()
    g, outs, _, _ = gpu_graph(spec, 0)
    ptr = g.eval(outs)[0]
    out = g.view(ptr, (configs.C2_ROWS, configs.C2_COLS))
    rng = np.random.default_rng(7)
    rows = np.sort(rng.choice(configs.C2_ROWS, 512, replace=False))
    rows[0], rows[-1] = 0, configs.C2_ROWS - 1
    got = out[torch.as_tensor(rows, device=out.device)].cpu().numpy()
    sub = configs.c2(rows=len(rows))
    og, oo = from_spec(sub)
    names = {n["name"]: n for n in spec["nodes"] if n["op"] in ("VAR", "CONST")}
    over = {}
    for n in og.nodes:
        if n.op == "VAR" or (n.op == "CONST" and n.name in ("c",)):
            full = names[n.name]
            val = materialise(full["data"], full["shape"], rows=rows)
            if n.op == "VAR":
                over[n.id] = val
            else:
                n.value = val
    vals = evaluate(og, leaf_values(og, over))
    assert normwise(got, vals[oo[0]]) <= 1e-5


# ---------------------------------------------------------------- reductions
@pytest.mark.parametrize("shape,a0,a1", [((4096, 10), 1, 2), ((4096, 1024), 0, 1), ((64, 28, 28, 6), 0, 3),
                                         ((3, 5, 7, 9), 1, 3), ((1 << 20,), 0, 1), ((7, 300001), 1, 2),
                                         ((2, 3), 0, 2)])
@pytest.mark.parametrize("op", ["SUM", "MAX"])
def test_reductions(shape, a0, a1, op):
    x = materialise({"kind": "uniform", "tag": "red", "lo": 0.5, "hi": 1.5}, shape)
    g = cg.Graph(0)
    v = g.var(shape)
    e = g.add_node("EXP", [v])           # fused elementwise prologue
    r = g.add_node(op, [e], a0=a0, a1=a1)
    g.plan_memory([r])
    g.assign(v, x)
    g.eval([r])
    og = OGraph()
    ov = og.add_leaf("VAR", shape)
    oe = og.add_node("EXP", [ov])
    orr = og.add_node(op, [oe], {"a0": a0, "a1": a1})
    ref = evaluate(og, {ov: x})[orr]
    assert normwise(g.read(r), ref) <= 1e-5


def test_integer_sum_exact():
    n = 4000
    x = np.arange(n, dtype=np.float32)
    g = cg.Graph(0)
    v = g.var([n])
    s = g.add_node("SUM", [v], a0=0, a1=1)
    g.plan_memory([s])
    g.assign(v, x)
    g.eval([s])
    assert float(g.read(s)[0]) == n * (n - 1) / 2


# ---------------------------------------------------------------- dot / conv / pool (integer-valued: exact)
def _run_single(op, shapes, attrs, lo=-4, hi=5, seed=0):
    rng = np.random.default_rng(seed)
    xs = [rng.integers(lo, hi, s).astype(np.float32) for s in shapes]
    g = cg.Graph(0)
    ids = [g.var(s) for s in shapes]
    o = g.add_node(op, ids, **attrs)
    g.plan_memory([o])
    for i, x in zip(ids, xs):
        g.assign(i, x)
    g.eval([o])
    og = OGraph()
    oids = [og.add_leaf("VAR", s) for s in shapes]
    oo = og.add_node(op, oids, attrs)
    ref = evaluate(og, dict(zip(oids, xs)))[oo]
    return g.read(o), ref


@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (200, 70, 33), (4096, 10, 1024), (5, 1024, 784)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_dot_integer_exact(m, n, k, ta, tb):
    sa = (k, m) if ta else (m, k)
    sb = (n, k) if tb else (k, n)
    got, ref = _run_single("DOT", [sa, sb], {"ta": ta, "tb": tb})
    assert np.array_equal(got, ref)


# shapes the tcgen05 path takes (16-byte row pitches), with ragged M / N / K tails
TC_SHAPES = [(128, 128, 32), (300, 136, 100), (129, 260, 36), (784, 1024, 512), (4096, 1024, 784),
             (40000, 512, 36),  # 128x256 tiles
             (1000, 48, 100), (500, 64, 64),  # 128x64 tiles
             (4100, 1024, 64), (19000, 256, 40)]  # CTA pairs with a ragged last 256-row tile


@pytest.mark.parametrize("m,n,k", TC_SHAPES)
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_dot_tc_integer_exact(m, n, k, ta, tb):
    """|x| <= 4 integers: hi == x, lo == 0 and every partial sum is exact in fp32,
    so the 3xTF32 tensor-core product must equal the f64 oracle bit for bit."""
    sa = (k, m) if ta else (m, k)
    sb = (n, k) if tb else (k, n)
    got, ref = _run_single("DOT", [sa, sb], {"ta": ta, "tb": tb})
    assert np.array_equal(got, ref)


# small-extent (HBM-bound SIMT) kernels and split-K tensor-core shapes of C3 / C4
SMALL_SHAPES = [(4096, 10, 1024), (1024, 10, 4096), (4096, 1024, 10), (84, 10, 8192), (8192, 84, 10),
                (300, 17, 33), (33, 300, 17), (120, 84, 8192), (400, 120, 8192), (7, 5, 3),
                (4097, 12, 1024), (513, 11, 130), (2049, 10, 20)]


@pytest.mark.parametrize("m,n,k", SMALL_SHAPES)
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_dot_small_and_splitk_integer_exact(m, n, k, ta, tb):
    sa = (k, m) if ta else (m, k)
    sb = (n, k) if tb else (k, n)
    got, ref = _run_single("DOT", [sa, sb], {"ta": ta, "tb": tb}, -2, 3)
    assert np.array_equal(got, ref)


def test_tf32_truncation_probe():
    """The production 3xTF32 path feeds the raw fp32 tile as the hi operand, relying
    on tcgen05.mma.kind::tf32 truncating fp32 inputs to TF32.  Check that against
    an explicitly masked hi tile: the two products must be bit-identical."""
    import ctypes
    import torch
    f = cg.lib().cgx_dot_tc
    f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int]
    torch.manual_seed(0)
    A = torch.rand(384, 512, device="cuda") * 2 - 1
    B = torch.rand(512, 256, device="cuda") * 2 - 1
    C0 = torch.zeros(384, 256, device="cuda")
    C1 = torch.zeros(384, 256, device="cuda")
    assert f(A.data_ptr(), B.data_ptr(), C0.data_ptr(), 384, 256, 512, 0, 0, None, 0) == 0
    assert f(A.data_ptr(), B.data_ptr(), C1.data_ptr(), 384, 256, 512, 0, 0, None, 1) == 0
    assert torch.equal(C0, C1)


@pytest.mark.parametrize("m,n,k", [(512, 384, 1000), (4096, 1024, 1024), (1024, 1024, 4096)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1)])
def test_dot_tc_float_3xtf32(m, n, k, ta, tb):
    """U[-1, 1) operands, 3xTF32 on tcgen05.  Error budget: the
    split itself is exact to ~2^-21 per product, but the tensor core's fp32
    accumulation does not round to nearest (measured on B200: 1.0e-5 normwise at
    K = 1000, i.e. ~1 ulp of |C| per MMA step, a truncation bias over 3*K/8 steps).
    A 1xTF32 product gives >= 1e-4 here (2^-11 per product), so 5e-5 still proves
    the lo terms are applied.  The analytic bound 3*ceil(K/8)*2^-23*max sum|a||b|
    / max|C| is asserted as well."""
    rng = np.random.default_rng(7)
    sa = (k, m) if ta else (m, k)
    sb = (n, k) if tb else (k, n)
    a = rng.uniform(-1, 1, sa).astype(np.float32)
    b = rng.uniform(-1, 1, sb).astype(np.float32)
    g = cg.Graph(0)
    va, vb = g.var(sa), g.var(sb)
    o = g.add_node("DOT", [va, vb], ta=ta, tb=tb)
    g.plan_memory([o])
    g.assign(va, a)
    g.assign(vb, b)
    g.eval([o])
    A = a.astype(np.float64).T if ta else a.astype(np.float64)
    B = b.astype(np.float64).T if tb else b.astype(np.float64)
    err = normwise(g.read(o), A @ B)
    ref = A @ B
    bound = 3 * -(-k // 8) * 2.0 ** -23 * float((np.abs(A) @ np.abs(B)).max()) / float(np.abs(ref).max())
    print(f"dot {m}x{n}x{k} ta={ta} tb={tb}: normwise {err:.3g} (analytic bound {bound:.3g})")
    assert err <= min(bound, 5e-5)


@pytest.mark.parametrize("sh,pad", [(1, 0), (1, 1), (2, 0), (2, 1)])
def test_conv_family_integer_exact(sh, pad):
    a = {"sh": sh, "sw": sh, "pad": pad}
    got, ref = _run_single("CONV2D", [(3, 11, 9, 4), (3, 5, 4, 6)], a, -3, 4)
    assert np.array_equal(got, ref)
    ho, wo = ref.shape[1], ref.shape[2]
    got, ref = _run_single("CONV2D_BWD_INPUT", [(3, ho, wo, 6), (3, 5, 4, 6)], dict(a, h=11, w=9), -3, 4)
    assert np.array_equal(got, ref)
    got, ref = _run_single("CONV2D_BWD_KERNEL", [(3, 11, 9, 4), (3, ho, wo, 6)], dict(a, kh=3, kw=5), -3, 4)
    assert np.array_equal(got, ref)


# C4's conv geometries (whole-image shared-memory kernels) and a wide-channel
# geometry that takes the generic kernels; every conv op, integer-valued => exact
CONV_CASES = [((8, 28, 28, 1), (5, 5, 1, 6), 1, 1), ((8, 14, 14, 6), (5, 5, 6, 16), 1, 0),
              ((4, 13, 11, 3), (3, 3, 3, 8), 2, 1), ((4, 12, 12, 5), (5, 3, 5, 20), 2, 0),
              ((4, 13, 11, 3), (3, 3, 3, 8), 1, 1), ((3, 9, 10, 12), (3, 3, 12, 16), 1, 0),
              ((2, 17, 15, 2), (5, 5, 2, 10), 1, 1), ((2, 15, 13, 6), (5, 5, 6, 8), 1, 1),
              ((2, 11, 12, 5), (3, 3, 5, 7), 1, 0),
              ((2, 9, 9, 40), (3, 3, 40, 48), 1, 1), ((2, 9, 9, 40), (3, 3, 40, 48), 2, 0)]

# geometries of C5's InceptionV3 convolutions (tcgen05 implicit GEMM, forward)
TC_CONV_CASES = [((2, 35, 35, 64), (3, 3, 64, 96), 1, 1), ((2, 35, 35, 32), (3, 3, 32, 64), 2, 0),
                 ((4, 17, 17, 48), (7, 1, 48, 64), 1, 1), ((2, 17, 17, 80), (1, 7, 80, 48), 1, 1),
                 ((2, 8, 8, 1280), (1, 1, 1280, 320), 1, 1), ((3, 15, 13, 12), (5, 5, 12, 20), 1, 1),
                 ((2, 31, 29, 3), (3, 3, 3, 32), 2, 0), ((2, 20, 20, 6), (5, 5, 6, 16), 1, 1),
                 ((2, 8, 8, 64), (3, 3, 64, 448), 1, 1), ((16, 35, 35, 32), (1, 1, 32, 512), 1, 1),
                 # CTA-pair tiles (>= one wave of 256-row units) on the 4-channel and element gathers
                 ((32, 35, 35, 20), (3, 3, 20, 128), 1, 1), ((128, 31, 29, 3), (3, 3, 3, 64), 2, 0),
                 # Ci % 32 == 0: TMA im2col tiles (SAME/VALID, strides 1/2, asymmetric SAME pads, 1xn / nx1 taps)
                 ((2, 17, 17, 32), (3, 3, 32, 64), 2, 1), ((3, 16, 16, 64), (3, 3, 64, 32), 2, 1),
                 ((2, 17, 17, 32), (1, 7, 32, 64), 1, 1), ((2, 17, 17, 32), (7, 1, 32, 64), 1, 1),
                 ((2, 12, 13, 96), (5, 5, 96, 48), 1, 1), ((9, 35, 35, 64), (3, 3, 64, 96), 1, 1),
                 ((4, 37, 33, 32), (3, 3, 32, 32), 2, 0),
                 # the InceptionV3 stem (Ci = 3, stride 2, VALID): the row-band kernel; 5 images
                 # cover full bands, the 5-row last band and a unit split across CTAs
                 ((5, 299, 299, 3), (3, 3, 3, 32), 2, 0),
                 # stem layers 2 / 3: input rows staged once in a ring (VALID 32 -> 32, SAME 32 -> 64)
                 ((3, 149, 149, 32), (3, 3, 32, 32), 1, 0), ((3, 147, 147, 32), (3, 3, 32, 64), 1, 1),
                 # Ci % 16 == 0: pairs of 16-channel im2col boxes; K % 32 == 16 exercises the zero half-slab
                 ((2, 12, 12, 16), (3, 3, 16, 32), 1, 1), ((2, 17, 17, 48), (5, 5, 48, 64), 1, 1),
                 ((2, 15, 15, 80), (3, 3, 80, 192), 1, 0), ((3, 16, 15, 48), (3, 3, 48, 64), 2, 1)]


@pytest.mark.parametrize("xs,ws,st,pad", TC_CONV_CASES)
def test_conv_tc_forward_integer_exact(xs, ws, st, pad):
    got, ref = _run_single("CONV2D", [xs, ws], {"sh": st, "sw": st, "pad": pad}, -2, 3)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("xs,ws,st,pad", TC_CONV_CASES[:3])
def test_conv_tc_forward_float(xs, ws, st, pad):
    """U[-1, 1) data: 3xTF32 implicit GEMM within the dot error budget."""
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, xs).astype(np.float32)
    w = rng.uniform(-1, 1, ws).astype(np.float32)
    g = cg.Graph(0)
    vx, vw = g.var(xs), g.var(ws)
    o = g.add_node("CONV2D", [vx, vw], sh=st, sw=st, pad=pad)
    g.plan_memory([o])
    g.assign(vx, x)
    g.assign(vw, w)
    g.eval([o])
    og = OGraph()
    ox, ow = og.add_leaf("VAR", xs), og.add_leaf("VAR", ws)
    oo = og.add_node("CONV2D", [ox, ow], {"sh": st, "sw": st, "pad": pad})
    assert normwise(g.read(o), evaluate(og, {ox: x, ow: w})[oo]) <= 5e-5


@pytest.mark.parametrize("xs,ws,st,pad", CONV_CASES)
def test_conv_geometries_integer_exact(xs, ws, st, pad):
    a = {"sh": st, "sw": st, "pad": pad}
    got, ref = _run_single("CONV2D", [xs, ws], a, -2, 3)
    assert np.array_equal(got, ref)
    ys = ref.shape
    got, ref = _run_single("CONV2D_BWD_INPUT", [ys, ws], dict(a, h=xs[1], w=xs[2]), -2, 3)
    assert np.array_equal(got, ref)
    got, ref = _run_single("CONV2D_BWD_KERNEL", [xs, ys], dict(a, kh=ws[0], kw=ws[1]), -2, 3)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("batch", [2400, 8192])
@pytest.mark.parametrize("xs,ws,pad", [((28, 28, 1), (5, 5, 1, 6), 1), ((14, 14, 6), (5, 5, 6, 16), 0)])
def test_c4_conv_geometries_at_batch(batch, xs, ws, pad):
    """C4's two convolutions at the batch sizes the bench runs (8192) and at one
    that leaves ragged per-block image chunks (2400): every conv op of the
    training graph, values in {-1, 0, 1} so every partial sum stays below 2^24
    and fp32 accumulation in any order is exact => bit-exact vs the oracle."""
    a = {"sh": 1, "sw": 1, "pad": pad}
    xs = (batch,) + xs
    got, ref = _run_single("CONV2D", [xs, ws], a, -1, 2, seed=batch)
    assert np.array_equal(got, ref)
    ys = ref.shape
    if ws[2] > 1:
        got, ref = _run_single("CONV2D_BWD_INPUT", [ys, ws], dict(a, h=xs[1], w=xs[2]), -1, 2, seed=batch + 1)
        assert np.array_equal(got, ref)
    got, ref = _run_single("CONV2D_BWD_KERNEL", [xs, ys], dict(a, kh=ws[0], kw=ws[1]), -1, 2, seed=batch + 2)
    assert np.array_equal(got, ref)


def test_maxpool_bwd_tiled_exact():
    """2x2/2 windows tiling a 28x28 input (the scatter kernel), ties included."""
    rng = np.random.default_rng(3)
    x = rng.integers(0, 3, (4, 28, 28, 6)).astype(np.float32)
    dy = rng.integers(1, 5, (4, 14, 14, 6)).astype(np.float32)
    a = {"kh": 2, "kw": 2, "sh": 2, "sw": 2, "pad": 0}
    g = cg.Graph(0)
    vx, vd = g.var(x.shape), g.var(dy.shape)
    o = g.add_node("MAXPOOL2D_BWD", [vx, vd], **a)
    g.plan_memory([o])
    g.assign(vx, x)
    g.assign(vd, dy)
    g.eval([o])
    og = OGraph()
    ox, od = og.add_leaf("VAR", x.shape), og.add_leaf("VAR", dy.shape)
    oo = og.add_node("MAXPOOL2D_BWD", [ox, od], a)
    assert np.array_equal(g.read(o), evaluate(og, {ox: x, od: dy})[oo])


@pytest.mark.parametrize("k,s,pad", [(2, 2, 0), (3, 2, 0), (3, 1, 1), (3, 2, 1), (8, 8, 0)])
@pytest.mark.parametrize("c", [4, 12, 32, 96])
def test_pools_channel_vectorised(k, s, pad, c):
    """C % 4 == 0: the float4-over-channels pool kernels (C5's pools)."""
    a = {"kh": k, "kw": k, "sh": s, "sw": s, "pad": pad}
    got, ref = _run_single("MAXPOOL2D", [(2, 17, 16, c)], a, -3, 4)
    assert np.array_equal(got, ref)
    got, ref = _run_single("AVGPOOL2D", [(2, 17, 16, c)], a, -3, 4)
    assert normwise(got, ref) <= 1e-6


@pytest.mark.parametrize("shape,s,pad", [((1, 9, 147, 64), 2, 0), ((3, 35, 35, 288), 1, 1), ((2, 17, 17, 768), 2, 0),
                                         ((2, 8, 8, 1280), 1, 1)])
def test_pools_c5_shapes(shape, s, pad):
    """C5's 3x3 pools (stride 2 VALID max, stride 1 SAME average) at their widths."""
    a = {"kh": 3, "kw": 3, "sh": s, "sw": s, "pad": pad}
    got, ref = _run_single("MAXPOOL2D", [shape], a, -3, 4)
    assert np.array_equal(got, ref)
    got, ref = _run_single("AVGPOOL2D", [shape], a, -3, 4)
    assert normwise(got, ref) <= 1e-6


def test_concat_vectorised():
    rng = np.random.default_rng(4)
    xs = [rng.standard_normal((2, 5, 3, c)).astype(np.float32) for c in (64, 96, 32, 128)]
    g = cg.Graph(0)
    ids = [g.var(x.shape) for x in xs]
    cat = g.add_node("CONCAT", ids, axis=3)
    g.plan_memory([cat])
    for i, x in zip(ids, xs):
        g.assign(i, x)
    g.eval([cat])
    assert np.array_equal(g.read(cat), np.concatenate(xs, axis=3))


@pytest.mark.parametrize("shape", [(3, 9, 9, 16), (2, 13, 13, 6), (2, 26, 26, 6), (2, 8, 9, 16)])
def test_maxpool2_few_channels_exact(shape):
    """C4's 2x2 stride-2 VALID max pools (C = 6, 16; odd sizes drop a row / column):
    forward and backward bit-identical to the oracle, with tied maxima."""
    rng = np.random.default_rng(5)
    a = {"kh": 2, "kw": 2, "sh": 2, "sw": 2, "pad": 0}
    x = rng.integers(0, 3, shape).astype(np.float32)
    ho, wo = shape[1] // 2, shape[2] // 2
    dy = rng.integers(1, 5, (shape[0], ho, wo, shape[3])).astype(np.float32)
    g = cg.Graph(0)
    vx, vd = g.var(x.shape), g.var(dy.shape)
    mp = g.add_node("MAXPOOL2D", [vx], **a)
    o = g.add_node("MAXPOOL2D_BWD", [vx, vd], **a)
    g.plan_memory([mp, o])
    g.assign(vx, x)
    g.assign(vd, dy)
    g.eval([mp, o])
    og = OGraph()
    ox, od = og.add_leaf("VAR", x.shape), og.add_leaf("VAR", dy.shape)
    omp = og.add_node("MAXPOOL2D", [ox], a)
    oo = og.add_node("MAXPOOL2D_BWD", [ox, od], a)
    vals = evaluate(og, {ox: x, od: dy})
    assert np.array_equal(g.read(mp), vals[omp])
    assert np.array_equal(g.read(o), vals[oo])


@pytest.mark.parametrize("k,s,pad", [(2, 2, 0), (3, 2, 0), (3, 1, 1), (3, 2, 1)])
def test_pools_exact(k, s, pad):
    a = {"kh": k, "kw": k, "sh": s, "sw": s, "pad": pad}
    got, ref = _run_single("MAXPOOL2D", [(2, 9, 8, 3)], a, 0, 3)
    assert np.array_equal(got, ref)
    ho, wo = ref.shape[1], ref.shape[2]
    rng = np.random.default_rng(1)
    x = rng.integers(0, 3, (2, 9, 8, 3)).astype(np.float32)
    dy = rng.integers(1, 5, (2, ho, wo, 3)).astype(np.float32)
    g = cg.Graph(0)
    vx, vd = g.var(x.shape), g.var(dy.shape)
    o = g.add_node("MAXPOOL2D_BWD", [vx, vd], **a)
    av = g.add_node("AVGPOOL2D", [vx], **a)
    g.plan_memory([o, av])
    g.assign(vx, x)
    g.assign(vd, dy)
    g.eval([o, av])
    og = OGraph()
    ox, od = og.add_leaf("VAR", x.shape), og.add_leaf("VAR", dy.shape)
    oo = og.add_node("MAXPOOL2D_BWD", [ox, od], a)
    oa = og.add_node("AVGPOOL2D", [ox], a)
    vals = evaluate(og, {ox: x, od: dy})
    assert np.array_equal(g.read(o), vals[oo])
    assert normwise(g.read(av), vals[oa]) <= 1e-6


def test_concat_reshape():
    rng = np.random.default_rng(2)
    xs = [rng.standard_normal((2, 3, 4, c)).astype(np.float32) for c in (5, 7, 2)]
    g = cg.Graph(0)
    ids = [g.var(x.shape) for x in xs]
    cat = g.add_node("CONCAT", ids, axis=3)
    r = g.add_node("RESHAPE", [cat], dims=[6, 56])
    n = g.add_node("NEG", [r])
    g.plan_memory([n])
    for i, x in zip(ids, xs):
        g.assign(i, x)
    g.eval([n])
    assert np.array_equal(g.read(n), -np.concatenate(xs, axis=3).reshape(6, 56))


# ---------------------------------------------------------------- random DAGs + incremental
@pytest.mark.parametrize("flags", MODES)
def test_random_graphs_and_incremental(flags):
    import random
    for seed in range(40):
        spec = random_spec(seed, simple_values=True)
        g, outs, _, _ = gpu_graph(spec, flags)
        og, oo = from_spec(spec)
        c = compile_graph(og, oo, flags)
        model = IncrementalModel(c)
        state = leaf_values(c.g)
        rng = random.Random(seed)
        vars_ = [v for v in c.gamma if c.g.nodes[v].op == "VAR"]
        for step in range(5):
            if vars_ and step and rng.random() < 0.7:
                x = rng.choice(vars_)
                val = materialise({"kind": "uniform", "tag": f"s{seed}_{step}", "lo": 0.5, "hi": 1.5},
                                  c.g.nodes[x].shape)
                state[x] = val
                g.assign(x, val)
                model.assign(x)
            ev = c.outputs if rng.random() < 0.7 else rng.sample(c.outputs, 1)
            g.eval(ev)
            model.eval(ev)
            ref = evaluate(c.g, state, ancestors(c.g, list(ev) + [u for u, _ in c.g.updates]))
            for o in ev:
                got = g.read(o)
                assert normwise(got, ref[o]) <= 2e-5, (seed, flags, step, o)
            for v in c.gamma:
                if v in model.count:
                    assert g.eval_count(v) == model.count[v], (seed, flags, step, v)
            for u, v in c.g.updates:
                state[v] = ref[u].copy()


def test_random_graphs_with_pow():
    """POW (numpy power semantics; powf on the GPU) inside random fused DAGs.
    Every POW node is made an output and checked against the oracle's POW applied
    to the GPU's own operand values (elementwise, <= 8 ulp relative; identical
    NaN / inf pattern), so the check isolates the op from the conditioning of
    the graph around it; graphs without DOT (whose cos / sin of large dot
    products amplify rounding by |argument|) are also checked end to end at the
    elementwise-graph tolerance."""
    from oracle.ops import eval_op
    n_pow = 0
    for seed in range(3000, 3040):
        spec = random_spec(seed, simple_values=True, extra_binary=("POW", "POW"), allow_updates=False)
        pows = [n for n in spec["nodes"] if n["op"] == "POW"]
        n_pow += len(pows)
        spec["outputs"] = list(spec["outputs"]) + [n["id"] for n in pows] + sorted(
            {p for n in pows for p in n["preds"] if spec["nodes"][p]["op"] not in ("VAR", "CONST")})
        g, outs, _, _ = gpu_graph(spec, 0)
        g.eval(outs)
        ref, og, _ = oracle_outputs(spec)
        leaves = leaf_values(og)
        for n in pows:
            a, b = [g.read(p) if p in outs else leaves[p] for p in n["preds"]]
            want = eval_op("POW", [a, b], {}, og.nodes[n["id"]].shape).astype(np.float64)
            got = g.read(n["id"]).astype(np.float64)
            assert np.array_equal(np.isnan(got), np.isnan(want)), (seed, n["id"])
            fin = np.isfinite(want)
            assert np.array_equal(np.isfinite(got), fin), (seed, n["id"])
            rel = np.abs(got[fin] - want[fin]) / np.maximum(np.abs(want[fin]), 1e-30)
            assert rel.size == 0 or rel.max() <= 8 * 2.0 ** -23, (seed, n["id"], rel.max())
        if not any(n["op"] == "DOT" for n in spec["nodes"]):
            for o in outs:
                assert normwise(g.read(o), ref[o]) <= 2e-5, (seed, o)
    assert n_pow >= 40


# ---------------------------------------------------------------- training graphs (10 iterations)
# Gate: the graph OUTPUTS (loss at every
# iteration, final logits) and the weight tensors at 1e-3 normwise.  A bias
# vector b = b0 - lr sum_it sum_s d_it[s] is a zero-initialised sum of
# mixed-sign, ReLU-masked per-sample terms: normwise it is ill-conditioned (a
# textbook fp32 sgemm in the oracle's place moves C3's b1 / b2 by 8.5e-3 /
# 1.4e-2), so biases are gated at 1e-3 RELATIVE TO THE SUMMATION'S CONDITION
# lr sum_it sum_s |d_it[s]| (max over components) — the componentwise error
# bound of a sum.  Measured for that fp32-sgemm stand-in: C3 b1/b2/b3 1.7e-4 /
# 2.6e-4 / 9.6e-6, C4 (batch 8192) <= 4e-5.  The final logits L = h.W + b are
# gated the same way, relative to max_ij (sum_k |h_ik||W_kj| + |b_j|) of the
# oracle's last iteration (the componentwise error bound of a dot + bias); their
# normwise error is printed.  Reason: at
# batch 8192 a ReLU decision on a value 3.6e-7 max|z| from the kink is taken
# differently at iteration 0 and the untrained network's dynamics amplify it
# ~1.4x per step (teacher-forced per-step logits error: 5e-6).
COND_TOL = 1e-3


def _train_parity(spec, iters, tol):
    g, outs, _, _ = gpu_graph(spec, 0)
    og, oo = from_spec(spec)
    per = {n["name"]: n["data"] for n in spec["nodes"] if n.get("name") in spec["meta"]["per_iteration"]}
    hist, state, cond = oracle_trajectory(og, oo, iters, per)
    name_to_id = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    for it in range(iters):
        for name, d in per.items():
            i = name_to_id[name]
            g.assign(i, materialise(retag(d, f"{d['tag']}@{it}"), spec["nodes"][i]["shape"]))
        g.eval(outs)
        loss = float(g.read(outs[0]).ravel()[0])
        ref = float(hist[it][oo[0]].ravel()[0])
        assert abs(loss - ref) <= tol * abs(ref), (it, loss, ref)
    errs = {}
    logits = g.read(outs[1])
    errs["logits (normwise)"] = normwise(logits, hist[-1][oo[1]])
    errs["logits"] = float(np.max(np.abs(logits.astype(np.float64) - hist[-1][oo[1]]))) / cond[oo[1]]
    assert errs["logits"] <= COND_TOL, errs
    for u, v in og.updates:
        name = og.nodes[v].name
        got = g.read(v)
        if v in cond:
            errs[name] = float(np.max(np.abs(got.astype(np.float64) - state[v]))) / cond[v]
            errs[name + " (normwise)"] = normwise(got, state[v])
            assert errs[name] <= COND_TOL, (name, errs)
        else:
            errs[name] = normwise(got, state[v])
            assert errs[name] <= tol, (name, errs)
    print(spec["name"], {k: f"{e:.2e}" for k, e in errs.items()})


def _teacher_forced(spec, iters, tol, rewrites=0):
    """Each iteration starts from the ORACLE's parameter state (cg_assign of every
    update target), so the comparison measures one evaluation + update_iopair per
    step instead of 10 steps of chaotic amplification.  The pre-activations
    (inputs of every RELU) are extra graph outputs: each is checked against the
    oracle, and everything downstream is compared with the oracle re-evaluated
    from the GPU's pre-activations, so a ReLU mask or max-pool argmax decision on
    a value within rounding of the kink (observed: C3 batch 256, iteration 9,
    |Z| = 2.3e-7 of max|Z|) is taken identically on both sides."""
    spec = dict(spec)
    # pinned: pre-activations (ReLU decisions) and the gradients entering the
    # optimiser (AdaGrad's lr*g/(sqrt(s)+eps) is a sign-like map of tiny g)
    pre = [n["preds"][0] for n in spec["nodes"] if n["op"] == "RELU"]
    grads = [n["id"] for n in spec["nodes"] if n["op"] == "ALLREDUCE_SUM"]
    zs = pre + grads
    spec["outputs"] = list(spec["outputs"]) + zs
    g, outs, _, _ = gpu_graph(spec, 0, rewrites=rewrites)
    og, oo = from_spec(spec)
    per = {n["name"]: n["data"] for n in spec["nodes"] if n.get("name") in spec["meta"]["per_iteration"]}
    name_to_id = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    state = leaf_values(og)
    needed = ancestors(og, list(oo) + [u for u, _ in og.updates])
    worst = 0.0
    for it in range(iters):
        for name, d in per.items():
            i = name_to_id[name]
            state[i] = materialise(retag(d, f"{d['tag']}@{it}"), spec["nodes"][i]["shape"])
            g.assign(i, state[i])
        for _, v in og.updates:
            g.assign(v, state[v])
        g.eval(outs)
        free = evaluate(og, state, needed)
        gz = {z: g.read(z) for z in zs}
        pinned = evaluate_pinned(og, state, gz, needed)
        # the gradients against the oracle pinned at the pre-activations only: every
        # ReLU mask and max-pool argmax (taken on relu(pre-activation)) is then the
        # GPU's, as this test's reading intends (compared with the free oracle, one
        # argmax within rounding of a tie moved a whole window's gradient: C4 batch
        # 64, iteration 1, after the conv2 kernel's k order changed)
        pinned_pre = evaluate_pinned(og, state, {z: gz[z] for z in pre}, needed)
        errs = [normwise(gz[z], free[z]) for z in pre]
        errs += [normwise(gz[z], pinned_pre[z]) for z in grads]
        errs += [normwise(g.read(o), pinned[o]) for o in oo if o not in gz]
        nxt = dict(state)
        apply_updates(og, pinned, nxt)
        errs += [normwise(g.read(v), nxt[v]) for _, v in og.updates]
        worst = max(worst, max(errs))
        assert max(errs) <= tol, (it, errs)
        apply_updates(og, free, state)
    print(spec["name"], f"teacher-forced worst normwise {worst:.2e}")


def test_c3_small_training():
    _teacher_forced(configs.c3(batch=256, widths=(784, 128, 64, 10)), 10, 1e-4)


def test_c3_full_training():
    """BASELINE configs[2] at full size (batch 4096, 784-1024-1024-10), 10 free-running iterations."""
    _train_parity(configs.c3(), 10, 1e-3)


def test_c4_small_training():
    _teacher_forced(configs.c4(batch=64), 10, 1e-4)


def test_c4_full_training():
    """BASELINE configs[3] at full size (batch 8192, the bench's launch
    configuration), 10 FREE-RUNNING iterations against the oracle: loss at every
    iteration, final logits and every weight at 1e-3 normwise, biases at 1e-3 of
    their summation condition (COND_TOL).  The oracle takes ~3 min of CPU."""
    _train_parity(configs.c4(), 10, 1e-3)


def test_c5_inception_sampled_images():
    """BASELINE configs[4] at full size: InceptionV3 at 299x299x3, batch 256, in the
    bench's launch configuration; the oracle evaluates images {0, 255} (inference is
    independent per image) and logits + softmax must agree to 1e-3 normwise."""
    spec = configs.c5()
    g, outs, rep, info = gpu_graph(spec, 0)
    assert info["pool_bytes"] < info["unshared_bytes"]
    g.eval(outs)
    logits, probs = g.read(outs[0]), g.read(outs[1])
    small = configs.c5(batch=2)
    og, oo = from_spec(small)
    xrec = spec["nodes"][0]
    assert xrec["name"] == "X"
    xs = materialise(xrec["data"], xrec["shape"], rows=[0, 255])
    vals = evaluate(og, leaf_values(og, {0: xs}))
    for i, row in enumerate([0, 255]):
        e_l = normwise(logits[row], vals[oo[0]][i])
        e_p = normwise(probs[row], vals[oo[1]][i])
        print(f"C5 image {row}: logits {e_l:.2e} softmax {e_p:.2e}")
        assert e_l <= 1e-3 and e_p <= 1e-3


@pytest.mark.parametrize("c", [96, 288, 320, 384, 1000])
def test_in_place_elementwise_group(c):
    """An elementwise group that slides onto its dying input's block (Alg. 1 in-place
    reuse) must read every element before any thread overwrites it: rows of
    width 288/320/384 give thread blocks that are not a multiple of the row width."""
    rng = np.random.default_rng(5)
    R = 4099
    x1 = rng.standard_normal((R, c // 2)).astype(np.float32)
    x2 = rng.standard_normal((R, c - c // 2)).astype(np.float32)
    g = cg.Graph(0)
    v1, v2 = g.var(x1.shape), g.var(x2.shape)
    cat = g.add_node("CONCAT", [v1, v2], axis=1)
    two = g.const(np.float32(2.0))
    one = g.const(np.float32(1.0))
    out = g.add_node("RELU", [g.add_node("SUB", [g.add_node("MUL", [cat, two]), one])])
    info = g.plan_memory([out])
    assert info["n_blocks"] == 1, "the elementwise group must slide onto the concat's block"
    g.assign(v1, x1)
    g.assign(v2, x2)
    for _ in range(3):
        g.eval([out], cg.EVAL_FULL)
        ref = np.maximum(np.concatenate([x1, x2], axis=1) * np.float32(2) - np.float32(1), 0)
        assert np.array_equal(g.read(out), ref)


# ---------------------------------------------------------------- f1 rewrites on the GPU
def test_c2_with_rewrites():
    """C2 with the paper's rewrites (3 FMAs): still the eager result within 1e-5."""
    spec = configs.c2(300, 1024)
    g, outs, rep, _ = gpu_graph(spec, 0, rewrites=cg.RW_ALL)
    assert rep["rw_fma"] == 3
    g.eval(outs)
    ref, _, _ = oracle_outputs(spec)
    assert normwise(g.read(outs[0]), ref[outs[0]]) <= 1e-5


def test_fused_adagrad_closed_form():
    """FusedAdagrad(lr=0.1, eps=1e-8)(g=1, s=4) = 0.1/(2+1e-8), computed in f64
    with one rounding on both sides: bit-exact."""
    g = cg.Graph(0)
    gv, sv = g.var([3]), g.var([3])
    lr, eps = g.const(np.float32(0.1)), g.const(np.float32(1e-8))
    d = g.add_node("DIV", [g.add_node("MUL", [lr, gv]), g.add_node("ADD", [g.add_node("SQRT", [sv]), eps])])
    g.set_rewrites(cg.RW_ADAGRAD)
    rep = g.optimise([d])
    assert rep["rw_adagrad"] == 1
    g.plan_memory([d])
    g.assign(gv, np.ones(3, np.float32))
    g.assign(sv, np.full(3, 4.0, np.float32))
    g.eval([d])
    want = np.float32(np.float64(np.float32(0.1)) * 1.0 / (2.0 + np.float64(np.float32(1e-8))))
    assert np.all(g.read(d) == want) and abs(float(want) - 0.05) < 1e-6


@pytest.mark.parametrize("flags", [0, cg.PLAN_NO_FUSION])
def test_random_graphs_with_rewrites(flags):
    for seed in range(40):
        spec = random_spec(seed, allow_updates=False, simple_values=True, rewrite_bait=True)
        g, outs, _, _ = gpu_graph(spec, flags, rewrites=cg.RW_ALL)
        g.eval(outs)
        ref, _, oo = oracle_outputs(spec)
        for o in oo:
            assert normwise(g.read(o), ref[o]) <= 2e-5, (seed, o)


def test_c3_adagrad_training_with_rewrites():
    """C3 with AdaGrad and every rewrite on (6 Fused_Adagrad + FMA nodes), teacher-forced."""
    _teacher_forced(configs.c3(batch=256, widths=(784, 128, 64, 10), optimizer="adagrad"), 10, 1e-4,
                    rewrites=cg.RW_ALL)


# ---------------------------------------------------------------- f2: epilogue fusion
def test_dot_bias_relu_epilogue_fusion_and_incremental():
    """DOT -> ADD(bias) -> SUB(scalar) -> RELU runs in the tensor-core epilogue
    (n_fused == 1) with the unfused kernels' exact per-op rounding; re-assigning
    only the bias still recomputes the pair (the DOT value is never materialised)."""
    rng = np.random.default_rng(21)
    M, N, K = 1000, 384, 200
    a = rng.integers(-3, 4, (M, K)).astype(np.float32)
    b = rng.integers(-3, 4, (K, N)).astype(np.float32)
    bias = rng.standard_normal((1, N)).astype(np.float32)
    g = cg.Graph(0)
    va, vb, vbias = g.var(a.shape), g.var(b.shape), g.var(bias.shape)
    half = g.const(np.float32(0.5))
    d = g.add_node("DOT", [va, vb], ta=0, tb=0)
    out = g.add_node("RELU", [g.add_node("SUB", [g.add_node("ADD", [d, vbias]), half])])
    info = g.plan_memory([out])  # (CG_PLAN_INCREMENTAL would pin d as a Var frontier: no fusion)
    assert info["n_fused"] == 1
    for x, v in ((va, a), (vb, b), (vbias, bias)):
        g.assign(x, v)
    g.eval([out])

    def ref(bias_):
        z = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
        return np.maximum((z + bias_) - np.float32(0.5), np.float32(0))
    assert np.array_equal(g.read(out), ref(bias))
    bias2 = rng.standard_normal((1, N)).astype(np.float32)
    g.assign(vbias, bias2)
    g.eval([out])
    assert np.array_equal(g.read(out), ref(bias2))
    assert g.eval_count(d) == 2


@pytest.mark.parametrize("xs,ws", [((16, 35, 35, 48), (3, 3, 48, 64)), ((16, 35, 35, 32), (1, 1, 32, 96))])
def test_conv_bn_relu_epilogue_fusion(xs, ws):
    """C5's conv -> BN (SUB mean, DIV sd, MUL gamma, ADD beta) -> RELU chain fused
    (enough output tiles that no split-K is needed: split-K convs are not fused)."""
    rng = np.random.default_rng(22)
    co = ws[3]
    spec_vals = {"x": rng.uniform(-1, 1, xs).astype(np.float32), "w": rng.uniform(-0.2, 0.2, ws).astype(np.float32)}
    mean = rng.uniform(-0.1, 0.1, (co,)).astype(np.float32)
    sd = rng.uniform(0.7, 1.2, (co,)).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, (co,)).astype(np.float32)
    beta = rng.uniform(-0.1, 0.1, (co,)).astype(np.float32)
    g = cg.Graph(0)
    vx, vw = g.var(xs), g.var(ws)
    cm, cs, cgm, cb = g.const(mean), g.const(sd), g.const(gamma), g.const(beta)
    y = g.add_node("CONV2D", [vx, vw], sh=1, sw=1, pad=1)
    t = g.add_node("ADD", [g.add_node("MUL", [g.add_node("DIV", [g.add_node("SUB", [y, cm]), cs]), cgm]), cb])
    out = g.add_node("RELU", [t])
    info = g.plan_memory([out])
    assert info["n_fused"] == 1
    g.assign(vx, spec_vals["x"])
    g.assign(vw, spec_vals["w"])
    g.eval([out])
    og = OGraph()
    ox, ow = og.add_leaf("VAR", xs), og.add_leaf("VAR", ws)
    oy = og.add_node("CONV2D", [ox, ow], {"sh": 1, "sw": 1, "pad": 1})
    yv = evaluate(og, {ox: spec_vals["x"], ow: spec_vals["w"]})[oy]
    want = np.maximum(((((yv - mean) / sd) * gamma) + beta).astype(np.float32), 0)
    assert normwise(g.read(out), want) <= 5e-5


def _run_training_state(spec, iters):
    g, outs, _, _ = gpu_graph(spec, 0)
    per = {n["name"]: n["data"] for n in spec["nodes"] if n.get("name") in spec["meta"]["per_iteration"]}
    name_to_id = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    for it in range(iters):
        for name, d in per.items():
            i = name_to_id[name]
            g.assign(i, materialise(retag(d, f"{d['tag']}@{it}"), spec["nodes"][i]["shape"]))
        g.eval(outs)
    vals = [g.read(o) for o in outs] + [g.read(i) for i in name_to_id.values()]
    g.destroy()
    return vals


@pytest.mark.parametrize("which", ["c3", "c4"])
def test_concurrent_capture_bit_identical(which, monkeypatch):
    """CG_STREAMS=4 captures independent groups on several streams (block-reuse,
    workspace and collective dependencies as graph edges).  The kernels and their
    internal summation orders are unchanged, so any missing dependency (a race)
    shows up as a bit difference against the one-stream Gamma order."""
    spec = configs.c3(batch=512, widths=(784, 256, 128, 10)) if which == "c3" else configs.c4(batch=128)
    monkeypatch.setenv("CG_STREAMS", "1")
    ref = _run_training_state(spec, 4)
    monkeypatch.setenv("CG_STREAMS", "4")
    got = _run_training_state(spec, 4)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- R14 zero-copy CONCAT
def test_zero_copy_concat_inception_block():
    """An Inception-style block: two tensor-core conv branches with a BN-like
    scale/shift + ReLU epilogue, a max-pool branch and a nested concat; the conv
    branches must store straight into their slices of the concat block (the
    epilogue's row stride = the concat's channels), the pool branch through a
    slice copy, and every value must match the oracle."""
    rng = np.random.default_rng(21)
    n, h, w, ci = 16, 35, 35, 32  # >= one wave of 128-row tiles: no split-K, the epilogue stores
    og = OGraph()
    g = cg.Graph(0)
    x = rng.uniform(-1, 1, (n, h, w, ci)).astype(np.float32)
    vx, ox = g.var(x.shape), og.add_leaf("VAR", x.shape)
    vals = {ox: x}
    branches_g, branches_o = [], []
    for k, co in enumerate((64, 96)):
        wk = (rng.uniform(-1, 1, (3, 3, ci, co)) / 9).astype(np.float32)
        sc = rng.uniform(0.5, 1.5, (co,)).astype(np.float32)
        sh = rng.uniform(-0.1, 0.1, (co,)).astype(np.float32)
        vw, ow = g.var(wk.shape), og.add_leaf("VAR", wk.shape)
        vs, os_ = g.const(sc), og.add_leaf("CONST", sc.shape, value=sc)
        vb, ob = g.const(sh), og.add_leaf("CONST", sh.shape, value=sh)
        vals[ow] = wk
        cv = g.add_node("CONV2D", [vx, vw], sh=1, sw=1, pad=1)
        cvo = og.add_node("CONV2D", [ox, ow], {"sh": 1, "sw": 1, "pad": 1})
        r = g.add_node("RELU", [g.add_node("ADD", [g.add_node("MUL", [cv, vs]), vb])])
        ro = og.add_node("RELU", [og.add_node("ADD", [og.add_node("MUL", [cvo, os_]), ob])])
        branches_g.append((r, vw, wk))
        branches_o.append(ro)
    mp = g.add_node("MAXPOOL2D", [vx], kh=3, kw=3, sh=1, sw=1, pad=1)
    mpo = og.add_node("MAXPOOL2D", [ox], {"kh": 3, "kw": 3, "sh": 1, "sw": 1, "pad": 1})
    inner = g.add_node("CONCAT", [branches_g[0][0], branches_g[1][0]], axis=3)
    inner_o = og.add_node("CONCAT", branches_o, {"axis": 3})
    cat = g.add_node("CONCAT", [inner, mp], axis=3)
    cat_o = og.add_node("CONCAT", [inner_o, mpo], {"axis": 3})
    out = g.add_node("NEG", [cat])
    out_o = og.add_node("NEG", [cat_o])
    g.plan_memory([out])
    g.assign(vx, x)
    for _, vw, wk in branches_g:
        g.assign(vw, wk)
    g.eval([out])
    st = g.view_stats()
    assert st["direct"] == 2 and st["copied"] == 1, st
    ref = evaluate(og, vals)[out_o]
    assert normwise(g.read(out), ref) <= 5e-5
    g.destroy()
