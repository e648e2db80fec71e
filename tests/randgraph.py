"""Seeded random graph specs for property tests (test input generation only).

Builds workloads-format specs with mixed broadcast shapes ([4,8], [1,8], [4,1],
[8], scalars), reductions, DOT, RESHAPE, and random update edges.  Shape
validity is checked by retrying with the oracle's Graph (test-side use).
"""
from __future__ import annotations

import random

from oracle.graph import Graph
from oracle.ops import CGError

UNARY = ["NEG", "ABS", "SQRT", "EXP", "LOG", "SIN", "COS", "TANH", "RELU"]
BINARY = ["ADD", "SUB", "MUL", "DIV", "MAX2", "MIN2", "RELU_GRAD"]
LEAF_SHAPES = [[4, 8], [1, 8], [4, 1], [8], []]


def random_spec(seed: int, n_ops=None, allow_updates=True, simple_values=False, rewrite_bait=False,
                extra_binary=()):
    rng = random.Random(seed)
    n_ops = n_ops if n_ops is not None else rng.randint(3, 40)
    nodes = []
    g = Graph()
    n_vars = rng.randint(1, 3)
    n_consts = rng.randint(0, 2)
    for k in range(n_vars):
        shp = rng.choice(LEAF_SHAPES[:4])
        lo, hi = (0.5, 1.5) if simple_values else (-1, 1)
        nodes.append({"id": len(nodes), "op": "VAR", "preds": [], "attrs": {}, "name": f"v{k}",
                      "shape": shp, "data": {"kind": "uniform", "tag": f"r{seed}v{k}", "lo": lo, "hi": hi}})
        g.add_leaf("VAR", shp)
    for k in range(n_consts):
        shp = rng.choice(LEAF_SHAPES)
        nodes.append({"id": len(nodes), "op": "CONST", "preds": [], "attrs": {}, "name": f"c{k}",
                      "shape": shp, "data": {"kind": "uniform", "tag": f"r{seed}c{k}", "lo": 0.5, "hi": 1.5}})
        g.add_leaf("CONST", shp)
    if rewrite_bait:  # exact 0 / 1 Consts and scalar Consts: identity / AdaGrad pattern material
        for k, (val, shp) in enumerate([(0.0, []), (1.0, []), (0.0, [4, 8]), (1.0, [1, 8])]):
            nodes.append({"id": len(nodes), "op": "CONST", "preds": [], "attrs": {}, "name": f"b{k}",
                          "shape": shp, "data": {"kind": "full", "value": val}})
            g.add_leaf("CONST", shp)
        nodes.append({"id": len(nodes), "op": "CONST", "preds": [], "attrs": {}, "name": "lr",
                      "shape": [], "data": {"kind": "literal", "values": [0.1]}})
        g.add_leaf("CONST", [])
        nodes.append({"id": len(nodes), "op": "CONST", "preds": [], "attrs": {}, "name": "eps",
                      "shape": [], "data": {"kind": "literal", "values": [1e-3]}})
        g.add_leaf("CONST", [])
    tries = 0
    made = 0
    while made < n_ops and tries < 50 * n_ops:
        tries += 1
        r = rng.random()
        ids = list(range(len(nodes)))
        # bias towards recent nodes so chains form
        def pick():
            if rng.random() < 0.6 and len(ids) > 3:
                return rng.choice(ids[-4:])
            return rng.choice(ids)
        if r < 0.35:
            op, preds, attrs = rng.choice(UNARY), [pick()], {}
        elif r < 0.75:
            a = pick()
            b = a if rng.random() < 0.1 else pick()
            op, preds, attrs = rng.choice(BINARY + list(extra_binary)), [a, b], {}
        elif r < 0.80:
            op, preds, attrs = "FMA", [pick(), pick(), pick()], {}
        elif r < 0.88:
            x = pick()
            rank = len(g.nodes[x].shape)
            if rank == 0:
                continue
            a0 = rng.randrange(rank)
            a1 = rng.randint(a0 + 1, rank)
            op, preds, attrs = rng.choice(["SUM", "MAX"]), [x], {"a0": a0, "a1": a1}
        elif r < 0.94:
            if rewrite_bait and rng.random() < 0.5:  # an AdaGrad adjusted-gradient pattern
                gv, sv = pick(), pick()
                lr = next(n["id"] for n in nodes if n.get("name") == "lr")
                eps = next(n["id"] for n in nodes if n.get("name") == "eps")
                try:
                    ids = []
                    for op_, pr in (("MUL", [lr, gv]), ("SQRT", [sv]), ("ADD", None), ("DIV", None)):
                        if op_ == "ADD":
                            pr = [ids[1], eps] if rng.random() < 0.5 else [eps, ids[1]]
                        if op_ == "DIV":
                            pr = [ids[0], ids[2]]
                        g.add_node(op_, pr, {})
                        nodes.append({"id": len(nodes), "op": op_, "preds": pr, "attrs": {}})
                        ids.append(len(nodes) - 1)
                    made += 4
                except CGError:
                    pass
                continue
            op, preds, attrs = "DOT", [pick(), pick()], {"ta": rng.randint(0, 1), "tb": rng.randint(0, 1)}
        else:
            x = pick()
            shp = g.nodes[x].shape
            n = 1
            for d in shp:
                n *= d
            dims = rng.choice([[n], [1, n], [n, 1]] + ([[8, 4], [2, 16]] if n == 32 else []))
            op, preds, attrs = "RESHAPE", [x], {"dims": dims}
        try:
            g.add_node(op, preds, attrs)
        except CGError:
            continue
        nodes.append({"id": len(nodes), "op": op, "preds": preds, "attrs": attrs})
        made += 1
    non_leaf = [n["id"] for n in nodes if n["op"] not in ("VAR", "CONST")]
    if not non_leaf:
        nodes.append({"id": len(nodes), "op": "NEG", "preds": [0], "attrs": {}})
        g.add_node("NEG", [0])
        non_leaf = [len(nodes) - 1]
    consumed = {p for n in nodes for p in n["preds"]}
    sinks = [i for i in non_leaf if i not in consumed]
    outs = rng.sample(sinks, min(len(sinks), rng.randint(1, 3)))
    if rng.random() < 0.3:
        outs.append(rng.choice(non_leaf))
    updates = []
    if allow_updates:
        for v in [n["id"] for n in nodes if n["op"] == "VAR"]:
            if rng.random() < 0.4:
                cands = [i for i in non_leaf if g.nodes[i].shape == g.nodes[v].shape]
                if cands:
                    updates.append([rng.choice(cands), v])
    return {"name": f"rand{seed}", "nodes": nodes, "outputs": outs, "updates": updates, "meta": {}}
