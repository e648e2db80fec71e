"""Fused AllReduce + update over peer memory (CG_PLAN_FUSED_COLL; SURVEY §8(f) f3,
P:26 "natural support for parallel and distributed computing").

One GPU is available, so the fused collective runs with world 1: every
ALLREDUCE_SUM group is the peer-memory kernel (coll.cu) with a sum over one rank,
and the SGD update that consumes it (W - lr * g) is evaluated inside that kernel
instead of in its own generated elementwise kernel.  The sum of one term is the
identity and the chain uses the generated kernels' IEEE per-op rounding, so the
training trajectory must be BIT-IDENTICAL to the plain plan, with every update
group fused away (n_fused) and fewer launches.  The independent collectives of
an executor step must have been issued as one batched launch.
"""
import ctypes

import numpy as np
import pytest

from paper_1812_03770_b200 import cg
from tests.gpu_util import leaf_data
from workloads import configs
from workloads.gen import materialise, retag

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _single_stream(monkeypatch):
    """These checks count launches, batched collectives and executor fusions of the
    default single-stream capture (CG_STREAMS > 1 issues collectives unbatched and
    leaves out the fusions whose side buffers the concurrent schedule cannot order)."""
    monkeypatch.delenv("CG_STREAMS", raising=False)


def _build(spec, flags=0, **kw):
    g = cg.Graph(0, **kw)
    for rec in spec["nodes"]:
        data = leaf_data(rec)
        if rec["op"] in ("VAR", "CONST"):
            g.add_node(rec["op"], (), dims=rec["shape"], **({"data": data} if data is not None else {}))
        else:
            g.add_node(rec["op"], rec["preds"], **rec.get("attrs", {}))
    for u, v in spec["updates"]:
        g.add_update(u, v)
    outs = spec["outputs"]
    g.optimise(outs)
    info = g.plan_memory(outs, flags)
    return g, outs, info


def _run(spec, g, outs, iters):
    ids = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    hist = []
    for it in range(iters):
        for nm in spec["meta"]["per_iteration"]:
            rec = spec["nodes"][ids[nm]]
            g.assign(ids[nm], materialise(retag(rec["data"], f"{rec['data']['tag']}@{it}"), rec["shape"]))
        g.eval(outs)
        hist.append([g.read(o) for o in outs])
    return hist, {u: g.read(v) for u, v in spec["updates"]}


@pytest.mark.parametrize("which", ["c3", "c4"])
def test_fused_allreduce_update_bit_identical(which):
    spec = configs.c3(batch=512, widths=(784, 256, 128, 10)) if which == "c3" else configs.c4(batch=128)
    n_ar = sum(1 for n in spec["nodes"] if n["op"] == "ALLREDUCE_SUM")
    g0, outs, info0 = _build(spec)
    h0, w0 = _run(spec, g0, outs, 4)
    l0 = g0.launch_count()
    g1, outs1, info1 = _build(spec, cg.PLAN_FUSED_COLL)
    h1, w1 = _run(spec, g1, outs1, 4)
    l1 = g1.launch_count()
    for a, b in zip(h0, h1):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    for k in w0:
        assert np.array_equal(w0[k], w1[k]), f"parameter {k}"
    # every SGD update group is evaluated inside its collective
    assert info1["n_fused"] - info0["n_fused"] == n_ar, (info0["n_fused"], info1["n_fused"], n_ar)
    assert info1["n_groups"] == info0["n_groups"]  # same plan (an executor choice)
    assert l1 < l0, (l0, l1)
    assert g1.coll_batches() >= 1  # independent collectives of one step: one launch
    print(which, "launches plain", l0, "fused", l1, "batched collective launches", g1.coll_batches())
    g0.destroy()
    g1.destroy()


def test_fused_coll_handle_and_connect_rules():
    """world 2 without an NCCL id: planning with the flag works (no communicator),
    the 128-byte handle is available, evaluation before cg_coll_connect is refused."""
    spec = configs.c3(batch=64, widths=(784, 32, 10))
    g, outs, _ = _build(spec, cg.PLAN_FUSED_COLL, rank=0, world=2, nccl_id=None)
    h = g.coll_handle()
    assert len(h) == 128 and any(h)
    with pytest.raises(cg.CGError) as e:
        g.eval(outs)
    assert e.value.code == "CG_E_STATE"
    with pytest.raises(cg.CGError) as e:
        g.coll_connect([h])  # wrong world
    assert e.value.code == "CG_E_ARG"
    g.destroy()
    # without the flag (and without NCCL) an ALLREDUCE at world 2 cannot be planned
    with pytest.raises(cg.CGError) as e:
        _build(spec, 0, rank=0, world=2, nccl_id=None)
    assert e.value.code == "CG_E_ARG"
