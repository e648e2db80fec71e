"""Computation graph G = (V, E, lambda, U) (ORACLE — test infrastructure only).

Definition 1: V vertices, E edges (u feeds v), lambda: V -> O with
Var in O, U update edges with lambda(v) = Var for every (u, v) in U; (V, E)
acyclic.  Ids are dense in creation order and preds must already exist, so
creation order is itself a topological order and acyclicity holds by
construction.  Multi-edges are allowed (x <- y * y).
"""
from __future__ import annotations

import copy

import numpy as np

from workloads.gen import SEED, materialise

from .ops import ARITY, ATTR_KEYS, LEAF, CGError, infer_shape, numel


class Node:
    __slots__ = ("id", "op", "preds", "attrs", "shape", "name", "data", "value")

    def __init__(self, id, op, preds, attrs, shape, name=None, data=None):
        self.id = id
        self.op = op
        self.preds = list(preds)
        self.attrs = attrs
        self.shape = tuple(int(d) for d in shape)
        self.name = name
        self.data = data      # workloads.gen data spec for leaves
        self.value = None     # fp32 ndarray for Const (materialised lazily / folded)

    @property
    def nbytes(self):
        return 4 * numel(self.shape)


def _norm_attrs(op, attrs):
    keys = ATTR_KEYS.get(op, ())
    out = {}
    for k in keys:
        if k not in attrs:
            raise CGError("CG_E_ARITY", f"{op} missing attribute {k}")
        v = attrs[k]
        out[k] = [int(d) for d in v] if k == "dims" else int(v)
    return out


class Graph:
    def __init__(self, seed: int = SEED):
        self.nodes: list[Node] = []
        self.updates: list[tuple[int, int]] = []
        self.seed = seed

    # -- construction (Operator layer) ---------------------------------
    def add_leaf(self, op, shape, name=None, data=None, value=None):
        if op not in LEAF:
            raise CGError("CG_E_ARITY", f"{op} is not a leaf")
        n = Node(len(self.nodes), op, [], {}, shape, name, data)
        if value is not None:
            n.value = np.array(value, dtype=np.float32).reshape(n.shape)
        self.nodes.append(n)
        return n.id

    def add_node(self, op, preds, attrs=None):
        """add_node: preds must exist, arity checked, shape inferred eagerly."""
        if op not in ARITY or op in LEAF:
            raise CGError("CG_E_ARITY", f"unknown or leaf op {op}")
        ar = ARITY[op]
        if (ar >= 0 and len(preds) != ar) or (ar < 0 and len(preds) < 1):
            raise CGError("CG_E_ARITY", f"{op} takes {ar} inputs, got {len(preds)}")
        for p in preds:
            if not (0 <= p < len(self.nodes)):
                raise CGError("CG_E_BAD_NODE", f"unknown predecessor {p}")
        a = _norm_attrs(op, attrs or {})
        shape = infer_shape(op, [self.nodes[p].shape for p in preds], a)
        n = Node(len(self.nodes), op, preds, a, shape)
        self.nodes.append(n)
        return n.id

    def add_update(self, u, var):
        """(u, v) in U requires lambda(v) = Var (Def. 1); copy semantics, shapes equal."""
        if not (0 <= u < len(self.nodes)) or not (0 <= var < len(self.nodes)):
            raise CGError("CG_E_BAD_NODE", "unknown node in update edge")
        if self.nodes[var].op != "VAR":
            raise CGError("CG_E_NOT_VAR", f"update target {var} is not a Var")
        if any(v == var for _, v in self.updates):
            raise CGError("CG_E_DUP_UPDATE", f"Var {var} already has an update edge")
        if self.nodes[u].shape != self.nodes[var].shape:
            raise CGError("CG_E_UPDATE_SHAPE", f"update {u}->{var} shape mismatch")
        self.updates.append((u, var))

    # -- helpers -------------------------------------------------------------------
    def const_value(self, i):
        n = self.nodes[i]
        assert n.op == "CONST"
        if n.value is None:
            n.value = materialise(n.data, n.shape, self.seed)
        return n.value

    def var_ids(self):
        return [n.id for n in self.nodes if n.op == "VAR"]

    def clone(self):
        g = Graph(self.seed)
        g.nodes = [copy.copy(n) for n in self.nodes]
        for n in g.nodes:
            n.preds = list(n.preds)
        g.updates = list(self.updates)
        return g


def from_spec(spec: dict, seed: int = SEED) -> tuple[Graph, list[int]]:
    """Build a Graph from a workloads.configs spec; returns (graph, declared outputs)."""
    g = Graph(seed)
    for rec in spec["nodes"]:
        if rec["op"] in LEAF:
            i = g.add_leaf(rec["op"], rec["shape"], rec.get("name"), rec.get("data"))
        else:
            i = g.add_node(rec["op"], rec["preds"], rec.get("attrs", {}))
        assert i == rec["id"], "spec ids must be dense creation order"
    for u, v in spec.get("updates", []):
        g.add_update(u, v)
    return g, list(spec.get("outputs", []))
