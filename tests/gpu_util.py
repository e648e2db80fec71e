"""Helpers for the GPU parity tests: build a workloads spec on the CUDA path
(through the C ABI) and on the oracle, with the same seeded inputs."""
from __future__ import annotations

import numpy as np

from oracle.eager import evaluate, leaf_values, run_iterations
from oracle.graph import from_spec
from paper_1812_03770_b200 import cg
from workloads.gen import materialise


def leaf_data(rec, seed=1812):
    if rec["op"] in ("VAR", "CONST"):
        return materialise(rec["data"], rec["shape"], seed)
    return None


def gpu_graph(spec, flags=0, optimise=True, device=0, rewrites=0):
    g, outs = cg.build_from_spec(spec, device=device, data_fn=leaf_data)
    if rewrites:
        g.set_rewrites(rewrites)
    rep = g.optimise(outs) if optimise else None
    info = g.plan_memory(outs, flags)
    return g, outs, rep, info


def normwise(got, ref):
    """E(g, o) = max|g - o| / max|o|; max|g| if o == 0."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(got), fin), "non-finite pattern differs"
    if not fin.any():
        return 0.0
    d = np.max(np.abs(got[fin] - ref[fin]))
    m = np.max(np.abs(ref[fin]))
    return float(d / m) if m > 0 else float(np.max(np.abs(got[fin])))


def oracle_outputs(spec, overrides=None):
    og, oo = from_spec(spec)
    vals = evaluate(og, leaf_values(og, overrides))
    return {o: vals[o] for o in oo}, og, oo


def evaluate_pinned(og, leaf_vals, pinned, needed=None):
    """The oracle's eager evaluation (oracle.ops.eval_op node by node, creation
    order) with the values of the nodes in ``pinned`` (id -> array) taken as given
    instead of computed.  Used to compare everything downstream of a ReLU / max-pool
    decision under the SAME decision the GPU took (the pinned values themselves are
    checked against the unpinned oracle separately)."""
    from oracle.ops import eval_op
    vals = dict(leaf_vals)
    for n in og.nodes:
        if n.op in ("VAR", "CONST"):
            if n.id not in vals:
                vals[n.id] = og.const_value(n.id) if n.op == "CONST" else np.zeros(n.shape, np.float32)
            continue
        if n.id in pinned:
            vals[n.id] = pinned[n.id]
            continue
        if needed is not None and n.id not in needed:
            continue
        vals[n.id] = eval_op(n.op, [vals[p] for p in n.preds], n.attrs, n.shape)
    return vals
