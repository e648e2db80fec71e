"""Optimiser: CSE -> CF -> DCE, each applied once (ORACLE — test infrastructure only).

"The Optimiser layer defines several structural patterns that can be
optimised or removed before any computation is performed".
- CF: "Nodes whose value only depends on constant nodes can be
  evaluated once and for all when the graph is created, and the constant
  nodes can be removed."  Readings: fold only the FRONTIER
  (const non-Const nodes that are roots or have a non-const consumer); the
  folded node keeps its id and becomes a Const; ALLREDUCE_SUM and Var are
  never constant; non-finite folded values are values, not errors.
- CSE (north-star extension; the paper's list is "non-exhaustive"):
  one pass in increasing id order; commutative canonicalisation for
  ADD/MUL/MAX2/MIN2; Vars never merge; user Consts merge by bytes; the
  lowest id is the representative.  CSE runs BEFORE CF, so
  folded Consts are never value-compared.
- DCE: delete non-Var nodes not reachable backwards from the roots.
"""
from __future__ import annotations

from .eager import ancestors
from .graph import Graph
from .ops import COMMUTATIVE, eval_op


def _attrs_key(attrs):
    return tuple(sorted((k, tuple(v) if isinstance(v, list) else v) for k, v in attrs.items()))


class OptResult:
    def __init__(self, g, outputs, rep, dead, folded, cse, cf, dce, rw_counts=None, rw_lists=None):
        self.g = g                # optimised graph (dead nodes kept in the table, marked in ``dead``)
        self.outputs = outputs    # outputs redirected through rep
        self.rep = rep            # CSE representative map old -> new
        self.dead = dead          # ids removed by CSE or DCE
        self.folded = folded      # ids turned into Const by CF
        self.report = {"cse_merged": cse, "cf_folded": cf, "dce_removed": dce}
        self.report.update(rw_counts or {"rw_identity": 0, "rw_zeroed": 0, "rw_fma": 0, "rw_adagrad": 0})
        self.rewrites = rw_lists  # None unless the f1 rewrites were requested

    def live(self):
        return [n.id for n in self.g.nodes if n.id not in self.dead]


def cse(g: Graph, dead: set) -> dict:
    rep, seen = {}, {}
    for n in g.nodes:
        if n.id in dead:
            continue
        n.preds = [rep.get(p, p) for p in n.preds]
        if n.op == "VAR":
            continue
        key = (n.op, _attrs_key(n.attrs), n.shape,
               tuple(sorted(n.preds)) if n.op in COMMUTATIVE else tuple(n.preds),
               g.const_value(n.id).tobytes() if n.op == "CONST" else None)
        if key in seen:
            rep[n.id] = seen[key]
            dead.add(n.id)
        else:
            seen[key] = n.id
    return rep


def constant_fold(g: Graph, dead: set, roots, compute_values=True) -> list:
    C = set()
    for n in g.nodes:
        if n.id in dead:
            continue
        if n.op == "CONST" or (n.op not in ("VAR", "ALLREDUCE_SUM") and n.preds
                               and all(p in C for p in n.preds)):
            C.add(n.id)
    consumers = {}
    for n in g.nodes:
        if n.id in dead:
            continue
        for p in n.preds:
            consumers.setdefault(p, set()).add(n.id)
    rootset = set(roots)
    frontier = [v for v in sorted(C) if g.nodes[v].op != "CONST"
                and (v in rootset or any(c not in C for c in consumers.get(v, ())))]
    values = {}
    if compute_values and frontier:
        # eager evaluation of the const cone, creation order, fresh value per node
        cone = ancestors(g, frontier)
        vals = {}
        for n in g.nodes:
            if n.id not in cone:
                continue
            if n.op == "CONST":
                vals[n.id] = g.const_value(n.id)
            else:
                vals[n.id] = eval_op(n.op, [vals[p] for p in n.preds], n.attrs, n.shape)
        values = {v: vals[v] for v in frontier}
    for v in frontier:
        n = g.nodes[v]
        n.op, n.preds, n.attrs = "CONST", [], {}
        n.data = None
        n.value = values.get(v)
    return frontier


def dce(g: Graph, dead: set, roots) -> int:
    live = ancestors(g, roots)
    removed = 0
    for n in g.nodes:
        if n.id not in dead and n.op != "VAR" and n.id not in live:
            dead.add(n.id)
            removed += 1
    return removed


def optimise(g: Graph, outputs, compute_values=True, rewrites=0) -> OptResult:
    """[rewrites (f1, oracle/rewrite.py) ->] CSE -> CF -> DCE.  ``rep`` maps every
    removed id (identity rewrite or CSE merge) to its final representative."""
    g = g.clone()
    dead = set()
    rw_rep, rw_counts, rw_lists = {}, None, None
    if rewrites:
        from .rewrite import rewrite
        rw_rep, rw_counts, rw_lists = rewrite(g, outputs, rewrites, dead)

    def rw(v):
        while v in rw_rep:
            v = rw_rep[v]
        return v
    outputs = [rw(o) for o in outputs]
    g.updates = [(rw(u), v) for u, v in g.updates]
    crep = cse(g, dead)
    rep = {v: crep.get(rw(v), rw(v)) for v in rw_rep}
    rep.update(crep)
    outs = [crep.get(o, o) for o in outputs]
    g.updates = [(crep.get(u, u), v) for u, v in g.updates]
    roots = outs + [u for u, _ in g.updates]
    folded = constant_fold(g, dead, roots, compute_values)
    removed = dce(g, dead, roots)
    return OptResult(g, outs, rep, dead, folded, len(crep), len(folded), removed, rw_counts, rw_lists)


def no_optimise(g: Graph, outputs) -> OptResult:
    """The raw graph as an OptResult (cg_plan_memory without cg_optimise)."""
    return OptResult(g.clone(), list(outputs), {}, set(), [], 0, 0, 0)
