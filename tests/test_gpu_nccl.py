"""The NCCL path of the ALLREDUCE_SUM node on one GPU.

Only one GPU is available to the build, so the collective runs on a 1-rank
NCCL communicator (cg_create with world 1 and a unique id): every AllReduce is
then a real ncclAllReduce captured in the evaluation's CUDA graph, issued in
the deferred batches of csrc/schedule.cpp (one ncclGroupStart/End each).  A sum
over one rank is the identity, so the training trajectory must be BIT-IDENTICAL
to the same graph without a communicator (where the node slides in place or
copies), and the collectives must have been batched.
"""
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


def _build(spec, nccl_id=None):
    g = cg.Graph(0, nccl_id=nccl_id)
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
    g.plan_memory(outs, 0)
    return g, outs


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
def test_one_rank_nccl_allreduce_bit_identical(which):
    spec = configs.c3(batch=512, widths=(784, 256, 128, 10)) if which == "c3" else configs.c4(batch=128)
    n_ar = sum(1 for n in spec["nodes"] if n["op"] == "ALLREDUCE_SUM")
    assert n_ar == len(spec["updates"])
    g0, outs = _build(spec)
    h0, w0 = _run(spec, g0, outs, 4)
    g1, outs1 = _build(spec, nccl_id=cg.nccl_unique_id())
    h1, w1 = _run(spec, g1, outs1, 4)
    for a, b in zip(h0, h1):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    for k in w0:
        assert np.array_equal(w0[k], w1[k])
    # every evaluation issued its AllReduces in batches, not one call per gradient
    assert g1.coll_batches() >= 1
    print(which, "collective batches per eval:", g1.coll_batches(), "for", n_ar, "AllReduce nodes")
    g0.destroy()
    g1.destroy()
