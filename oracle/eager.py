"""Eager evaluation — the numeric definition every optimisation must reproduce
(ORACLE — test infrastructure only).

"The main idea behind a computation graph is to replace eager evaluation of
variables ... by the building of a graph": the graph's outputs equal
plain eager evaluation of its ops in any topological order.  So this
evaluates every node in creation order (a valid topological order)
into a FRESH allocation per node, computing in f64 and rounding once
to fp32 per node (ops.eval_op).  Update edges are applied after
an evaluation with parallel-assignment semantics: all sources are read as of
the end of the evaluation, then copied into their Var.
"""
from __future__ import annotations

import numpy as np

from workloads.gen import materialise, retag

from .graph import Graph
from .ops import eval_op


def leaf_values(g: Graph, overrides=None, seed=None):
    """Initial values of every leaf: Consts from their data spec, Vars from theirs
    unless ``overrides`` (id -> array) supplies one."""
    overrides = overrides or {}
    vals = {}
    for n in g.nodes:
        if n.op == "CONST":
            vals[n.id] = g.const_value(n.id)
        elif n.op == "VAR":
            if n.id in overrides:
                vals[n.id] = np.array(overrides[n.id], np.float32).reshape(n.shape)
            else:
                vals[n.id] = materialise(n.data, n.shape, g.seed if seed is None else seed)
    return vals


def evaluate(g: Graph, leaf_vals: dict, needed=None, dtype=np.float32) -> dict:
    """One eager evaluation.  ``leaf_vals``: id -> fp32 array for every Var/Const.
    ``needed``: optional set of ids to evaluate (others skipped); default all nodes."""
    vals = dict(leaf_vals)
    for n in g.nodes:
        if n.op in ("VAR", "CONST"):
            if n.id not in vals:
                vals[n.id] = g.const_value(n.id) if n.op == "CONST" else np.zeros(n.shape, np.float32)
            continue
        if needed is not None and n.id not in needed:
            continue
        vals[n.id] = eval_op(n.op, [vals[p] for p in n.preds], n.attrs, n.shape, dtype)
    return vals


def ancestors(g: Graph, roots) -> set:
    seen = set()
    stack = list(roots)
    while stack:
        v = stack.pop()
        if v in seen:
            continue
        seen.add(v)
        stack.extend(g.nodes[v].preds)
    return seen


def apply_updates(g: Graph, vals: dict, var_state: dict):
    """update_iopair: (u, v) in U simultaneously: value(v) <- copy(value(u))."""
    staged = [(v, np.array(vals[u], copy=True)) for u, v in g.updates]
    for v, x in staged:
        var_state[v] = x


def run_iterations(g: Graph, outputs, n_iter: int, per_iteration: dict | None = None,
                   var_init: dict | None = None):
    """Evaluate ``n_iter`` iterations with update edges, as a training loop does.

    ``per_iteration``: Var name -> data spec; iteration ``it`` assigns the spec
    retagged "<tag>@<it>" (SURVEY §8(d) tags).  Returns (list of {output id ->
    value} per iteration, final Var state)."""
    state = leaf_values(g, var_init)
    name_to_id = {n.name: n.id for n in g.nodes if n.op == "VAR"}
    needed = ancestors(g, list(outputs) + [u for u, _ in g.updates])
    hist = []
    for it in range(n_iter):
        if per_iteration:
            for name, spec in per_iteration.items():
                i = name_to_id[name]
                state[i] = materialise(retag(spec, f"{spec['tag']}@{it}"), g.nodes[i].shape, g.seed)
        vals = evaluate(g, state, needed)
        hist.append({o: vals[o] for o in outputs})
        apply_updates(g, vals, state)
    return hist, state
