"""Ordering gamma, Var signatures and fusion grouping (ORACLE — test infrastructure only).

gamma: "The topological ordering gamma we use for allocation and evaluation is
given by traversing the graph from the outputs using a post-order DFS"
(Def. 2).  Roots are the outputs in declaration order, then the
update sources in add_update order (reading R10); predecessors are
visited left to right; each node is emitted once.

Fusion grouping (motivated by "reduce memory access",
P:273, and "each vertex can only be computed once"): in reverse gamma,
an elementwise node joins the group of its consumers when all its consumers
lie in ONE group whose domain equals its shape; reductions start a group and
may only be its sink; every other op is a singleton group.
"""
from __future__ import annotations

from .ops import EW, LEAF, RED, numel

FLAG_INCREMENTAL = 1
FLAG_NO_FUSION = 2


def gamma(g, roots):
    """Iterative post-order DFS from ``roots``."""
    order, seen = [], set()
    for r in roots:
        if r in seen:
            continue
        seen.add(r)
        stack = [[r, 0]]
        while stack:
            top = stack[-1]
            preds = g.nodes[top[0]].preds
            if top[1] < len(preds):
                p = preds[top[1]]
                top[1] += 1
                if p not in seen:
                    seen.add(p)
                    stack.append([p, 0])
            else:
                order.append(top[0])
                stack.pop()
    return order


def consumers_in(g, nodes):
    """Distinct in-graph consumers of each node among ``nodes``."""
    cons = {v: [] for v in nodes}
    for v in nodes:
        for p in g.nodes[v].preds:
            if v not in cons[p]:
                cons[p].append(v)
    return cons


def descendants(g, order, x):
    """D(x): strict descendants of x within the planned node set ``order``."""
    inside = set(order)
    cons = consumers_in(g, order)
    out, stack = set(), [x]
    while stack:
        v = stack.pop()
        for c in cons.get(v, ()):
            if c in inside and c not in out:
                out.add(c)
                stack.append(c)
    return out


def signatures_and_frontier(g, order, update_targets):
    """CG_PLAN_INCREMENTAL rules 1-2: for every Var x in gamma that
    is not an update target, F(x) = {u not in D(x) u {x} : u has a consumer in D(x)}
    and sig(v) = {x : v in D(x)}."""
    sig = {v: set() for v in order}
    frontier = set()
    cons = consumers_in(g, order)
    for x in order:
        if g.nodes[x].op != "VAR" or x in update_targets:
            continue
        D = descendants(g, order, x)
        for v in D:
            sig[v].add(x)
        for u in order:
            if u == x or u in D:
                continue
            if any(c in D for c in cons[u]):
                frontier.add(u)
    return {v: frozenset(s) for v, s in sig.items()}, frontier


class Group:
    __slots__ = ("sink", "members", "domain", "inputs", "materialised", "safe", "kind")

    def __init__(self, sink, domain, kind):
        self.sink = sink
        self.members = [sink]
        self.domain = domain
        self.kind = kind
        self.inputs = []
        self.materialised = []
        self.safe = False

    def as_dict(self):
        return {"inputs": list(self.inputs), "materialised": list(self.materialised),
                "members": list(self.members), "sink": self.sink}


def group_nodes(g, order, keep, flags, sig=None):
    """c6-algo.  Returns groups in Gamma order (sorted by the gamma rank of the sink)."""
    rank = {v: i for i, v in enumerate(order)}
    cons = consumers_in(g, order)
    group_of = {}
    groups = []
    incremental = bool(flags & FLAG_INCREMENTAL)
    for v in reversed(order):
        n = g.nodes[v]
        if n.op in LEAF:
            continue
        if (flags & FLAG_NO_FUSION) or (n.op not in EW and n.op not in RED):
            G = Group(v, None, "op")
        elif n.op in RED:
            G = Group(v, g.nodes[n.preds[0]].shape, "red")
        else:
            cg = []
            for c in cons[v]:
                if group_of[c] not in cg:
                    cg.append(group_of[c])
            if (len(cg) == 1 and cg[0].domain is not None and n.shape == cg[0].domain
                    and (not incremental or sig[v] == sig[cg[0].sink])):
                cg[0].members.append(v)
                group_of[v] = cg[0]
                continue
            G = Group(v, n.shape, "ew")
        groups.append(G)
        group_of[v] = G
    groups.sort(key=lambda G: rank[G.sink])
    for G in groups:
        G.members.sort(key=lambda m: rank[m])
        mem = set(G.members)
        for m in G.members:
            for p in g.nodes[m].preds:
                if p not in mem and p not in G.inputs:
                    G.inputs.append(p)
        G.materialised = [m for m in G.members if m == G.sink or m in keep]
        ops = [g.nodes[m].op for m in G.members]
        G.safe = all(o in EW for o in ops) or (len(ops) == 1 and ops[0] in ("RESHAPE", "ALLREDUCE_SUM"))
    return groups, group_of


def dom_numel(g, G):
    return numel(g.nodes[G.sink].shape)
