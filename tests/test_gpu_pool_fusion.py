"""f2 fusion around C4's few-channel convolutions and 2x2 max pools, and full-tensor
operands in the GEMM epilogue (
P:273 "reduce memory access").

The executor computes an elementwise group inside a neighbouring kernel that is not
a GEMM: the bias ADD in the tcgen05 conv epilogue (conv_img_tc), the RELU in the
max pool that consumes it (a prologue: the pool reads the ADD's value, writes the
RELU's and pools it), and RELU_GRAD in the max-pool backward kernel (an epilogue
with a full-tensor operand, the forward pre-activation).  Each op keeps the
generated kernels' IEEE per-op rounding, so the training trajectory must be
BIT-IDENTICAL to the plan without these fusions, with six groups fewer launched.
"""
import os

import numpy as np
import pytest

from paper_1812_03770_b200 import cg
from tests.test_gpu_fused_coll import _build, _run
from workloads import configs
from workloads.gen import materialise, retag

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _single_stream(monkeypatch):
    """These checks count launches, batched collectives and executor fusions of the
    default single-stream capture (CG_STREAMS > 1 issues collectives unbatched and
    leaves out the fusions whose side buffers the concurrent schedule cannot order)."""
    monkeypatch.delenv("CG_STREAMS", raising=False)


def _build_env(spec, env, flags=0):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: v for k, v in env.items() if v is not None})
    try:
        return _build(spec, flags)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("batch,flags", [(128, 0), (96, cg.PLAN_FUSED_COLL), (8192, 0)])
def test_c4_pool_and_conv_fusion_bit_identical(batch, flags):
    spec = configs.c4(batch=batch)
    iters = 2 if batch > 1000 else 4
    g0, outs, info0 = _build_env(spec, {"CG_NO_POOL_FUSION": "1"}, flags)
    h0, w0 = _run(spec, g0, outs, iters)
    l0 = g0.launch_count()
    g1, outs1, info1 = _build(spec, flags)
    h1, w1 = _run(spec, g1, outs1, iters)
    l1 = g1.launch_count()
    # (the fused bias gradient sums in another fixed order: b1 and what follows
    # from it agree to rounding; everything else is bit-identical)
    for a, b in zip(h0, h1):
        for x, y in zip(a, b):
            assert np.allclose(x, y, rtol=1e-5, atol=1e-6)
    for k in w0:
        assert np.allclose(w0[k], w1[k], rtol=1e-5, atol=1e-6), f"parameter {k}"
    # conv1 / conv2 bias ADD, the two RELUs before the pools, the two RELU_GRADs after
    # the pool backward passes, RELU_GRAD(a3, dh3) in the dh3 GEMM's epilogue (a
    # full-tensor operand), db1 = SUM(da1) from conv1's backward-kernel dy reads, and
    # da1 itself formed inside that kernel from dp1 and the pool's codes
    nf = info1["n_fused"] - info0["n_fused"]
    assert nf == 9, (info0["n_fused"], info1["n_fused"])
    assert info1["n_groups"] == info0["n_groups"]
    assert l0 - l1 == nf * iters, (l0, l1)
    g0.destroy()
    g1.destroy()


def test_pool_prologue_with_operands_and_odd_sizes():
    """A longer prologue chain (SUB scalar, MUL column, MAX2 full tensor, RELU) into a
    2x2 pool and its backward with a RELU_GRAD epilogue, bit-equal to the unfused
    plan; an odd-sized pool (skipped last row / column) is not fused."""
    rng = np.random.default_rng(5)
    for hw, fused in ((12, 2), (13, 0)):
        x = rng.standard_normal((6, hw, hw, 16)).astype(np.float32)
        m = rng.standard_normal((6, hw, hw, 16)).astype(np.float32)
        colv = rng.standard_normal((16,)).astype(np.float32)
        dyv = rng.standard_normal((6, hw // 2, hw // 2, 16)).astype(np.float32)
        res = []
        for env in ({"CG_NO_POOL_FUSION": "1"}, {}):
            old = os.environ.pop("CG_NO_POOL_FUSION", None)
            os.environ.update(env)
            try:
                g = cg.Graph(0)
                vx, vm, vdy = g.var(x.shape), g.var(m.shape), g.var(dyv.shape)
                vc = g.const(colv)
                a = g.add_node("ADD", [vx, vm])  # the pre-activation (materialised: two consumers)
                t = g.add_node("MUL", [g.add_node("SUB", [a, g.const(np.float32(0.25))]), vc])
                h = g.add_node("RELU", [g.add_node("MAX2", [t, vm])])
                p = g.add_node("MAXPOOL2D", [h], kh=2, kw=2, sh=2, sw=2, pad=0)
                dh = g.add_node("MAXPOOL2D_BWD", [h, vdy], kh=2, kw=2, sh=2, sw=2, pad=0)
                da = g.add_node("RELU_GRAD", [a, dh])
                outs = [p, da]
                info = g.plan_memory(outs)
                for v, d in ((vx, x), (vm, m), (vdy, dyv)):
                    g.assign(v, d)
                g.eval(outs)
                res.append(([g.read(o) for o in outs], info["n_fused"]))
                g.destroy()
            finally:
                os.environ.pop("CG_NO_POOL_FUSION", None)
                if old is not None:
                    os.environ["CG_NO_POOL_FUSION"] = old
        (r0, n0), (r1, n1) = res
        for u, v in zip(r0, r1):
            assert np.array_equal(u, v), hw
        assert n1 - n0 == fused, (hw, n0, n1)
        # and the values themselves (numpy, same per-op fp32 rounding)
        a_ = x + m
        h_ = np.maximum(np.maximum((a_ - np.float32(0.25)) * colv, m), 0)
        n, H, W, C = h_.shape
        ho, wo = H // 2, W // 2
        win = h_[:, :2 * ho, :2 * wo].reshape(n, ho, 2, wo, 2, C)
        assert np.array_equal(r1[0], win.max(axis=(2, 4)))


def test_c3_relu_grad_in_gemm_epilogue_bit_identical():
    """C3's backward: dh_k = da_{k+1} . W^T feeds only RELU_GRAD(a_k, dh_k); a
    tensor-core GEMM's epilogue applies it with a_k read at [row, col] (a full-tensor
    operand), so dh_k never reaches HBM -- same values as the separate kernel."""
    spec = configs.c3(batch=512, widths=(784, 256, 128, 10))
    g0, outs, info0 = _build_env(spec, {"CG_NO_POOL_FUSION": "1"})
    h0, w0 = _run(spec, g0, outs, 4)
    g1, outs1, info1 = _build(spec)
    h1, w1 = _run(spec, g1, outs1, 4)
    for a, b in zip(h0, h1):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    for k in w0:
        assert np.array_equal(w0[k], w1[k]), f"parameter {k}"
    # dh1 (a tensor-core GEMM) takes it; dh2 = dL . W3^T (K = 10) is a SIMT small-K dot
    assert info1["n_fused"] - info0["n_fused"] == 1, (info0["n_fused"], info1["n_fused"])
    g0.destroy()
    g1.destroy()


def test_pool_codes_bit_identical_and_incremental():
    """2x2 max-pool backward reading the forward's recorded window decisions (one
    byte per output element) instead of the input: C4 trajectories are bit-identical
    to the plan without codes; asking for the backward value alone after the input
    changed still re-runs the forward (its decisions must be current)."""
    spec = configs.c4(batch=96)
    g0, outs, _ = _build_env(spec, {"CG_NO_POOL_CODES": "1"})
    h0, w0 = _run(spec, g0, outs, 3)
    g1, outs1, _ = _build(spec)
    h1, w1 = _run(spec, g1, outs1, 3)
    for a, b in zip(h0, h1):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    for k in w0:
        assert np.array_equal(w0[k], w1[k]), f"parameter {k}"
    g0.destroy()
    g1.destroy()

    rng = np.random.default_rng(9)
    shp = (4, 12, 12, 16)
    g = cg.Graph(0)
    vx, vdy = g.var(shp), g.var((4, 6, 6, 16))
    h = g.add_node("RELU", [vx])
    p = g.add_node("MAXPOOL2D", [h], kh=2, kw=2, sh=2, sw=2, pad=0)
    dh = g.add_node("MAXPOOL2D_BWD", [h, vdy], kh=2, kw=2, sh=2, sw=2, pad=0)
    g.plan_memory([p, dh], cg.PLAN_INCREMENTAL)
    dyv = rng.standard_normal((4, 6, 6, 16)).astype(np.float32)
    g.assign(vdy, dyv)

    def ref(xv):
        hv = np.maximum(xv, 0)
        win = hv.reshape(4, 6, 2, 6, 2, 16).transpose(0, 1, 3, 2, 4, 5).reshape(4, 6, 6, 4, 16)
        best = np.argmax(win, axis=3)  # first maximum, as the kernels
        out = np.zeros((4, 6, 6, 4, 16), np.float32)
        np.put_along_axis(out, best[:, :, :, None, :], dyv[:, :, :, None, :], axis=3)
        return out.reshape(4, 6, 6, 2, 2, 16).transpose(0, 1, 3, 2, 4, 5).reshape(shp)
    for it in range(3):
        xv = rng.standard_normal(shp).astype(np.float32)
        g.assign(vx, xv)
        g.eval([dh] if it else [p, dh])
        assert np.array_equal(g.read(dh), ref(xv)), it
    g.destroy()


def test_c4_fused_gradients_under_partial_demand():
    """Incremental evaluation through the executor fusions: after a new X, asking
    only for dW1 (whose dy, da1, is never materialised -- formed from dp1 and the
    pool's codes) or only for db1 (fused into the same kernel) must recompute the
    chain that feeds it (pool forward codes included) and match a full evaluation."""
    spec = configs.c4(batch=64)
    ids = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    grads = [n["id"] for n in spec["nodes"] if n["op"] == "CONV2D_BWD_KERNEL"]
    sums = [n["id"] for n in spec["nodes"] if n["op"] == "SUM" and n.get("attrs", {}).get("a1") == 3]
    want_nodes = grads + sums
    spec = dict(spec)
    spec["outputs"] = list(spec["outputs"]) + want_nodes
    g, outs, info = _build(spec)
    ref, _, _ = _build(spec)
    xrec = spec["nodes"][ids["X"]]
    for it in range(3):
        xv = materialise(retag(xrec["data"], f"X@pd{it}"), xrec["shape"])
        for gr in (g, ref):
            gr.assign(ids["X"], xv)
        ref.eval(outs, cg.EVAL_NO_UPDATE)
        for node in want_nodes:  # one output at a time, each after a fresh X on g
            g.assign(ids["X"], xv)
            g.eval([node], cg.EVAL_NO_UPDATE)
            assert np.array_equal(g.read(node), ref.read(node)), (it, node)
    g.destroy()
    ref.destroy()


def test_epilogue_division_bit_identical_to_separate_kernel():
    """The fused chains' DIV (C5's batch-norm x / sd) uses a branch-free Newton
    quotient when every operand of a 16-value group is in range and __fdiv_rn
    otherwise: the fused DOT epilogue equals the separate elementwise kernel bit for
    bit, also with zeros, huge / tiny magnitudes and infinities in the data."""
    rng = np.random.default_rng(17)
    M, N, K = 640, 192, 96
    a = rng.standard_normal((M, K)).astype(np.float32)
    a[::7, :] *= np.float32(1e25)   # quotients out of the fast path's range
    a[3, :] = 0.0
    b = rng.standard_normal((K, N)).astype(np.float32)
    sd = rng.uniform(0.5, 2.0, (N,)).astype(np.float32)
    sd[5] = np.float32(1e-30)
    sd[9] = np.float32(np.inf)
    mean = rng.standard_normal((N,)).astype(np.float32)
    res = []
    for env in ({"CG_NO_EPILOGUE_FUSION": "1"}, {}):
        old = os.environ.pop("CG_NO_EPILOGUE_FUSION", None)
        os.environ.update(env)
        try:
            g = cg.Graph(0)
            va, vb = g.var(a.shape), g.var(b.shape)
            d = g.add_node("DOT", [va, vb], ta=0, tb=0)
            out = g.add_node("RELU", [g.add_node("DIV", [g.add_node("SUB", [d, g.const(mean)]), g.const(sd)])])
            info = g.plan_memory([out])
            g.assign(va, a)
            g.assign(vb, b)
            g.eval([out])
            res.append((g.read(out), info["n_fused"]))
            g.destroy()
        finally:
            os.environ.pop("CG_NO_EPILOGUE_FUSION", None)
            if old is not None:
                os.environ["CG_NO_EPILOGUE_FUSION"] = old
    (r0, n0), (r1, n1) = res
    assert n1 == n0 + 1
    assert np.array_equal(r0.view(np.uint32), r1.view(np.uint32))
