"""Sibling 1x1 convolutions merged into one tensor-core GEMM (
P:273 "reduce memory access").

Inception blocks apply several 1x1 convolutions to the same input.  The executor
runs such siblings as ONE GEMM over their concatenated weights with a
column-routed epilogue: every column is still the same K-long 3xTF32 dot product
in the same order and each segment's chain uses its own per-column operands, so
the outputs must be BIT-IDENTICAL to the unmerged plan.  Merged members count in
n_fused.  Const weights are concatenated once at planning; Var weights may be
re-assigned between evaluations, so their concatenation is a launch of every
evaluation, which the second check covers (all weights, then one member's).
"""
import copy
import os

import numpy as np
import pytest

from paper_1812_03770_b200 import cg
from tests.gpu_util import leaf_data
from workloads import configs
from workloads.gen import materialise

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _single_stream(monkeypatch):
    """The merge is made for the single-stream capture only."""
    monkeypatch.delenv("CG_STREAMS", raising=False)


def _graph(spec, merge):
    old = os.environ.get("CG_NO_SIBLING_GEMM")
    if merge:
        os.environ.pop("CG_NO_SIBLING_GEMM", None)
    else:
        os.environ["CG_NO_SIBLING_GEMM"] = "1"
    try:
        g, outs = cg.build_from_spec(spec, device=0, data_fn=leaf_data)
        g.optimise(outs)
        info = g.plan_memory(outs, 0)
    finally:
        if old is None:
            os.environ.pop("CG_NO_SIBLING_GEMM", None)
        else:
            os.environ["CG_NO_SIBLING_GEMM"] = old
    return g, outs, info


def _pointwise_weights(spec):
    by_id = {r["id"]: r for r in spec["nodes"]}
    ws = []
    for r in spec["nodes"]:
        if r["op"] == "CONV2D":
            w = by_id[r["preds"][1]]
            if w["op"] in ("VAR", "CONST") and list(w["shape"][:2]) == [1, 1]:
                ws.append(w)
    return ws


def _with_var_weights(spec):
    """The same graph with the 1x1 weights as Vars (re-assignable)."""
    spec = copy.deepcopy(spec)
    ids = {w["id"] for w in _pointwise_weights(spec)}
    for r in spec["nodes"]:
        if r["id"] in ids:
            r["op"] = "VAR"
    return spec


@pytest.mark.parametrize("batch", [4, 32])
def test_c5_sibling_gemm_const_weights(batch):
    """C5 as configured (Const weights, concatenated once at planning)."""
    spec = configs.c5(batch=batch)
    res, nf = [], []
    for merge in (False, True):
        g, outs, info = _graph(spec, merge)
        try:
            g.eval(outs, cg.EVAL_SYNC)
            res.append([g.read(o) for o in outs])
            nf.append(info["n_fused"])
        finally:
            g.destroy()
    assert nf[1] - nf[0] >= 3, nf  # the blocks' sibling sets merged
    for x, y in zip(*res):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("batch", [4, 32])
def test_c5_sibling_gemm_var_weights(batch):
    spec = _with_var_weights(configs.c5(batch=batch))
    res = []
    nf = []
    for merge in (False, True):
        g, outs, info = _graph(spec, merge)
        try:
            g.eval(outs, cg.EVAL_SYNC)
            first = [g.read(o) for o in outs]
            # re-assign every 1x1 weight: the merged GEMM must see the new values
            for k, w in enumerate(_pointwise_weights(spec)):
                g.assign(w["id"], 0.5 * materialise(w["data"], w["shape"], 77 + k))
            g.eval(outs, cg.EVAL_SYNC)
            second = [g.read(o) for o in outs]
            # one member's weight alone (incremental evaluation: the merged launch
            # must re-run when any sibling's input changed)
            w = _pointwise_weights(spec)[1]
            g.assign(w["id"], -materialise(w["data"], w["shape"], 99))
            g.eval(outs, cg.EVAL_SYNC)
            third = [g.read(o) for o in outs]
        finally:
            g.destroy()
        res.append((first, second, third))
        nf.append(info["n_fused"])
    assert nf[1] - nf[0] >= 3, nf  # the blocks' sibling sets merged
    (f0, s0, t0), (f1, s1, t1) = res
    for a, b in ((f0, f1), (s0, s1), (t0, t1)):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    # each re-assignment changed the result (the checks above are not vacuous)
    assert any(not np.array_equal(x, y) for x, y in zip(f1, s1))
    assert any(not np.array_equal(x, y) for x, y in zip(s1, t1))
