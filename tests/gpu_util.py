"""Helpers for the GPU parity tests: build a workloads spec on the CUDA path
(through the C ABI) and on the oracle, with the same seeded inputs."""
from __future__ import annotations

import numpy as np

from oracle.eager import ancestors, apply_updates, evaluate, leaf_values
from oracle.graph import from_spec
from paper_1812_03770_b200 import cg
from workloads.gen import materialise, retag


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


def _bias_gradient_inputs(og):
    """For every SGD update edge (u, v): u = SUB(v, MUL(g, lr)) with g =
    [ALLREDUCE_SUM](SUM(d, axes)) — the bias pattern of configs._sgd — return
    {v: (d id, axes, lr id)}.  Weight updates (g = DOT) are not listed."""
    out = {}
    for u, v in og.updates:
        n = og.nodes[u]
        if n.op != "SUB" or n.preds[0] != v:
            continue
        m = og.nodes[n.preds[1]]
        if m.op != "MUL":
            continue
        g, lr = m.preds
        gn = og.nodes[g]
        if gn.op == "ALLREDUCE_SUM":
            gn = og.nodes[gn.preds[0]]
        if gn.op != "SUM":
            continue
        out[v] = (gn.preds[0], tuple(range(gn.attrs["a0"], gn.attrs["a1"])), lr)
    return out


def oracle_trajectory(og, oo, iters, per):
    """run_iterations with one extra output per bias parameter: the conditioning
    denominator of its 10-step SGD sum, lr * sum_it sum_samples |d_it| (the
    componentwise condition number of summation: a bias b = b0 - lr sum_it
    sum_s d_it[s] is only determined to rounding RELATIVE to this sum, and a
    ReLU / max-pool decision taken differently on a value within rounding of
    the kink moves b by one sample's term).  Returns (hist, state, cond)."""
    state = leaf_values(og)
    name_to_id = {n.name: n.id for n in og.nodes if n.op == "VAR"}
    needed = ancestors(og, list(oo) + [u for u, _ in og.updates])
    bias = _bias_gradient_inputs(og)
    cond = {v: 0.0 for v in bias}
    hist = []
    for it in range(iters):
        for name, spec in per.items():
            i = name_to_id[name]
            state[i] = materialise(retag(spec, f"{spec['tag']}@{it}"), og.nodes[i].shape, og.seed)
        vals = evaluate(og, state, needed)
        hist.append({o: vals[o] for o in oo})
        last = vals
        for v, (d, axes, lr) in bias.items():
            lrv = abs(float(np.asarray(vals[lr], np.float64).ravel()[0]))
            cond[v] = cond[v] + lrv * np.sum(np.abs(vals[d].astype(np.float64)), axis=axes)
        apply_updates(og, vals, state)
    cond = {v: float(np.max(c)) for v, c in cond.items()}
    # logits L = ADD(DOT(h, W), b): the summation condition of the last iteration's
    # logits, max_ij (sum_k |h_ik| |W_kj| + |b_j|) (componentwise bound of a dot + bias)
    for o in oo:
        n = og.nodes[o]
        if n.op == "ADD" and og.nodes[n.preds[0]].op == "DOT":
            dn = og.nodes[n.preds[0]]
            h = np.abs(last[dn.preds[0]].astype(np.float64))
            w = np.abs(last[dn.preds[1]].astype(np.float64))
            h = h.T if dn.attrs.get("ta") else h
            w = w.T if dn.attrs.get("tb") else w
            cond[o] = float(np.max(h @ w + np.abs(last[n.preds[1]].astype(np.float64))))
    return hist, state, cond
