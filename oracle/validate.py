"""Brute-force plan validator (ORACLE — test infrastructure only).

validate_plan: "recomputes lifetimes by brute force and reports
any block shared by overlapping lifetimes, any undersized block, any
keep-flagged node whose block is later reassigned".  Lifetimes are measured
in group steps t = index in Gamma: value a lives from def(a) to last(a) = the
last group reading it (infinity if kept).  Two values may share a
block only if one's lifetime ends before the other's starts, or it ends AT
that group, the group is in-place safe ("sliding"), and the two
have the same numel so element i maps to element i (R5, R13).
"""
from __future__ import annotations

import math

from .ops import numel


def lifetimes(c):
    """Per value: def = group step that writes it, last = last group step reading it.
    A zero-copy CONCAT family (R14: the root and its views share one block by
    design) is one lifetime: from its first def to the root's last read."""
    g = c.g
    d, last = {}, {}
    for t, G in enumerate(c.groups):
        for m in G.materialised:
            d[m] = t
        for p in G.inputs:
            last[p] = t
    for m in d:
        if m in c.keep_all:
            last[m] = math.inf
        else:
            last.setdefault(m, d[m])
    views = getattr(c.plan, "views", {})
    for v, spec in views.items():
        root = spec[0]
        if root in d and v in d:
            d[root] = min(d[root], d[v])
    for v, spec in views.items():
        root = spec[0]
        if root in d and v in d:
            d[v], last[v] = d[root], last[root]
    return d, last


def validate_plan(c, block=None, size=None):
    """Return a list of violation strings (empty = ok).  ``block``/``size`` may
    override the plan's (to test the validator on adversarial plans)."""
    g = c.g
    block = dict(c.plan.block if block is None else block)
    size = list(c.plan.size if size is None else size)
    d, last = lifetimes(c)
    errs = []
    materialised = [m for G in c.groups for m in G.materialised]
    for m in materialised:
        if m not in block:
            errs.append(f"value {m} has no block")
            continue
        if size[block[m]] < 4 * numel(g.nodes[m].shape):
            errs.append(f"undersized: block {block[m]} < value {m}")
    by_block = {}
    for m in materialised:
        if m in block:
            by_block.setdefault(block[m], []).append(m)
    # a zero-copy CONCAT family (R14) is represented by its root: the views share the
    # root's block and lifetime by construction
    views = getattr(c.plan, "views", {})
    for b, vs in by_block.items():
        vs = [v for v in vs if v not in views]
        for i in range(len(vs)):
            for j in range(len(vs)):
                a, bb = vs[i], vs[j]
                if a == bb or d[a] > d[bb]:
                    continue
                if d[a] == d[bb]:
                    if a < bb:
                        errs.append(f"values {a} and {bb} of one group share block {b}")
                    continue
                # d[a] < d[bb]
                if last[a] < d[bb]:
                    continue
                G = c.groups[d[bb]]
                if (last[a] == d[bb] and G.safe and a in G.inputs
                        and numel(g.nodes[a].shape) == numel(g.nodes[bb].shape)):
                    continue
                errs.append(f"overlap: {a} (live {d[a]}..{last[a]}) and {bb} (def {d[bb]}) share block {b}")
    return errs
