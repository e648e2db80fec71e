"""Host-compiler pipeline and canonical JSON dumps (ORACLE — test infrastructure only).

The structural products (rewritten graph, groups, memory plan) are algorithm
outputs that the C++ host compiler must reproduce BIT-EXACTLY; both sides
emit the same canonical JSON (sorted keys, no whitespace, integers and
op-name strings only; SURVEY §8(c) "Canonical dumps").
"""
from __future__ import annotations

import json

from .ops import LEAF, numel
from .optimise import no_optimise, optimise
from .planner import plan_memory
from .schedule import FLAG_INCREMENTAL, gamma, group_nodes, signatures_and_frontier


def canon(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


class Compiled:
    """Everything cg_optimise + cg_plan_memory decide, for one graph."""

    def __init__(self, raw, opt, outputs, flags):
        g = opt.g
        self.raw, self.opt, self.g, self.flags = raw, opt, g, flags
        self.outputs = [opt.rep.get(o, o) for o in outputs]
        self.roots = self.outputs + [u for u, _ in g.updates]
        self.gamma = gamma(g, self.roots)
        self.rank = {v: i for i, v in enumerate(self.gamma)}
        update_targets = {v for _, v in g.updates}
        self.sig, frontier = signatures_and_frontier(g, self.gamma, update_targets)
        keep = set(self.roots)
        if flags & FLAG_INCREMENTAL:
            keep |= frontier
        self.keep_all = keep
        self.external = {v for v in self.gamma if g.nodes[v].op in LEAF}
        self.keep = sorted(v for v in keep if v not in self.external)
        self.groups, self.group_of = group_nodes(g, self.gamma, keep, flags, self.sig)
        self.plan = plan_memory(g, self.groups, keep, flags)
        self.unshared_bytes = sum(4 * numel(n.shape) for n in raw.nodes if n.op not in LEAF)


def compile_graph(g, outputs, flags=0, do_optimise=True, compute_values=True, rewrites=0) -> Compiled:
    opt = optimise(g, outputs, compute_values, rewrites) if do_optimise else no_optimise(g, outputs)
    return Compiled(g, opt, outputs, flags)


def graph_json(opt) -> str:
    g = opt.g
    nodes = []
    for n in g.nodes:
        if n.id in opt.dead:
            continue
        nodes.append({"attrs": dict(n.attrs), "id": n.id, "op": n.op, "preds": list(n.preds),
                      "shape": list(n.shape)})
    d = {"dead": sorted(opt.dead), "folded": sorted(opt.folded), "nodes": nodes,
         "rep": [[k, opt.rep[k]] for k in sorted(opt.rep)]}
    if opt.rewrites is not None:
        d["rewrites"] = {k: sorted(v) for k, v in opt.rewrites.items()}
    return canon(d)


def plan_json(c: Compiled) -> str:
    p = c.plan
    return canon({"block": [[v, p.block[v]] for v in sorted(p.block)],
                  "block_bytes": list(p.size),
                  "gamma": list(c.gamma),
                  "groups": [G.as_dict() for G in c.groups],
                  "keep": list(c.keep),
                  "plan_bytes": p.plan_bytes, "pool_bytes": p.pool_bytes,
                  "unshared_bytes": c.unshared_bytes,
                  "views": [[v] + list(p.views[v]) for v in sorted(p.views)]})
