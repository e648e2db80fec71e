"""Incremental re-evaluation model and block-simulated evaluator (ORACLE — test infrastructure only).

"natural support for incremental computation (recomputation of exactly what
is needed when some input is modified)"; "If after evaluating it once,
we only modify the value of x3, there is no need to re-evaluate x2".
The paper never reconciles this with block sharing, so the engine
semantics are SURVEY §8(c) c9 (reading in DESIGN.md):

  valid(p)   := p external, or (not dirty[p] and owner[block[p]] == p)
  assign(x)  :  dirty[n] <- true for n in D(x)
  eval(outs) :  roots = outs + update sources (unless NO_UPDATE);
                R = demand-driven recompute set, closed under the clobber
                fix-point; launch R in Gamma order; owner/dirty/eval_count;
                update copy; dirty[D(v)] for every update target v.

``BlockSim`` executes a plan on simulated blocks (numpy arrays sized in
bytes), reading group inputs FROM BLOCKS, so any plan or recompute-set error
surfaces as a wrong value against fresh eager evaluation (the brute-force pin).
"""
from __future__ import annotations

import numpy as np

from .ops import eval_op, numel
from .schedule import descendants

EVAL_NO_UPDATE = 1


class IncrementalModel:
    def __init__(self, c):
        self.c = c
        g = c.g
        self.X = set(c.external)
        self.block = c.plan.block
        self.members = {v for G in c.groups for v in G.members}
        self.dirty = {v: True for v in self.members}
        self.owner = {}
        self.count = {v: 0 for v in c.gamma}
        self.D = {x: descendants(g, c.gamma, x) for x in c.gamma if g.nodes[x].op == "VAR"}
        self.gidx = {}
        for i, G in enumerate(c.groups):
            for m in G.members:
                self.gidx[m] = i

    def valid(self, p):
        return p in self.X or (not self.dirty[p] and self.owner.get(self.block[p]) == p)

    def assign(self, x):
        for n in self.D.get(x, ()):
            if n in self.dirty:
                self.dirty[n] = True

    def recompute_set(self, outs, flags=0):
        c = self.c
        roots = list(outs) + ([] if flags & EVAL_NO_UPDATE else [u for u, _ in c.g.updates])
        R = set()

        def demand(v, force=False):
            if v in self.X or self.gidx[v] in R:
                return
            if self.valid(v) and not force:
                return
            R.add(self.gidx[v])
            for p in c.groups[self.gidx[v]].inputs:
                demand(p)

        for r in roots:
            demand(r)
        while True:
            sim = dict(self.owner)
            bad = None
            for i, G in enumerate(c.groups):
                if i not in R:
                    continue
                for p in G.inputs:
                    if p not in self.X and sim.get(self.block[p]) != p:
                        bad = p
                        break
                if bad is not None:
                    break
                for m in G.materialised:
                    sim[self.block[m]] = m
            if bad is None:
                for r in roots:
                    if r not in self.X and sim.get(self.block[r]) != r:
                        bad = r
                        break
            if bad is None:
                break
            demand(bad, force=True)
        return R, roots

    def commit(self, R, flags=0):
        c = self.c
        for i in sorted(R):
            G = c.groups[i]
            for m in G.materialised:
                self.owner[self.block[m]] = m
            for n in G.members:
                self.dirty[n] = False
                self.count[n] += 1
        if not flags & EVAL_NO_UPDATE:
            for _, v in c.g.updates:
                self.assign(v)

    def eval(self, outs, flags=0):
        R, roots = self.recompute_set(outs, flags)
        self.commit(R, flags)
        return R


class BlockSim:
    """Run a compiled graph on simulated blocks with the incremental model."""

    def __init__(self, c, leaf_vals):
        self.c = c
        self.model = IncrementalModel(c)
        self.ext = {v: np.array(leaf_vals[v], np.float32) for v in c.external}
        self.blocks = [np.full(s // 4, np.nan, np.float32) for s in c.plan.size]

    def assign(self, x, value):
        self.ext[x] = np.array(value, np.float32).reshape(self.c.g.nodes[x].shape)
        self.model.assign(x)

    def read(self, v):
        if v in self.ext:
            return self.ext[v]
        n = self.c.g.nodes[v]
        return self.blocks[self.c.plan.block[v]][:numel(n.shape)].reshape(n.shape)

    def eval(self, outs, flags=0):
        c = self.c
        R, roots = self.model.recompute_set(outs, flags)
        for i in sorted(R):
            G = c.groups[i]
            local = {p: self.read(p).copy() for p in G.inputs}
            for m in G.members:
                n = c.g.nodes[m]
                local[m] = eval_op(n.op, [local[p] for p in n.preds], n.attrs, n.shape)
            for m in G.materialised:
                blk = self.blocks[c.plan.block[m]]
                blk[:numel(c.g.nodes[m].shape)] = local[m].ravel()
        self.model.commit(R, flags)
        result = {o: self.read(o).copy() for o in outs}
        if not flags & EVAL_NO_UPDATE:
            staged = [(v, self.read(u).copy()) for u, v in c.g.updates]
            for v, x in staged:
                self.ext[v] = x
        return result, R
