"""Memory plan: Algorithm 1 applied to fusion groups (ORACLE — test infrastructure only).

Algorithm 1 "Memory Allocation for CPU devices" with the prose
rules of P:316-320 and the caveats of P:294-297, read as R1-R13:
  R1  grow the largest block in *reusable* (prose P:319; not "in block")
  R2  the returned block leaves reusable
  R3  reusable.add(p) means "add block[p]"
  R4  keep = outputs + update sources (+ Var-frontier under CG_PLAN_INCREMENTAL);
      Var/Const are external
  R5  in-place preference = restriction inside best-fit to released inputs of
      equal numel
  R6  in-place-unsafe groups allocate before release
  R7  refs count distinct consuming groups (== edge multiplicity at node level)
  R8  ties -> lowest block id
  R9  sizes are exact bytes (numel*4); 256 B alignment only in the layout
  R11 the recursive Initialise is the post-order walk of gamma
  R13 in a safe (elementwise) group only inputs whose numel equals the group's
      domain may be released before allocation; broadcast (smaller) inputs are
      released after it, so no thread overwrites an element another thread
      still has to read.
  R14 zero-copy CONCAT ("reduce memory access"; a
      sub-block view, the offset != 0 extension of P:303-310): outside
      CG_PLAN_INCREMENTAL, an input v of a CONCAT c is planned as a VIEW of c's
      block when v is the sink of its own group, c's group is v's only consumer,
      v occurs once among c's inputs, v is not kept and v is not a Var / Const /
      RESHAPE / ALLREDUCE_SUM.  Element (o, i) of v (o over the axes before the
      concat axis, i within) is element o * inner(root) + offset + i of the view
      root.  Concats are visited outer-first (reverse Gamma), so a view CONCAT's
      inputs become views of the same root (offsets add).  The root's block is
      allocated when the first value of its family is (FindBestBlock, no in-place
      preference); views neither allocate nor release.
"""
from __future__ import annotations

from .ops import LEAF, numel
from .schedule import FLAG_INCREMENTAL, dom_numel

NO_VIEW_PRODUCERS = ("RESHAPE", "ALLREDUCE_SUM")

ALIGN = 256


def align_up(x, a=ALIGN):
    return (x + a - 1) // a * a


class Plan:
    def __init__(self):
        self.views = {}        # value id -> (root, outer, inner_root, offset, inner) (R14)
        self.block = {}        # value id -> block id
        self.size = []         # block id -> bytes (final, after growth)
        self.offsets = []
        self.pool_bytes = 0
        self.plan_bytes = 0


def find_best_block(reusable: set, size: list, s: int, pref=frozenset()):
    """FindBestBlock(s) (R1, R2, R5, R8).  Returns (block, created?)."""
    C = [b for b in reusable if size[b] >= s]
    if C:
        cand = [b for b in C if b in pref] or C
        b = min(cand, key=lambda b: (size[b], b))
    elif reusable:
        b = max(reusable, key=lambda b: (size[b], -b))
        size[b] = s
    else:
        size.append(s)
        return len(size) - 1, True
    reusable.remove(b)
    return b, False


def concat_views(g, groups, keep, flags):
    """R14: value -> (root, outer, inner_root, offset, inner) for zero-copy CONCAT."""
    if flags & FLAG_INCREMENTAL:
        return {}
    sink_of = {G.sink for G in groups}
    consumers = {}
    for G in groups:
        for p in G.inputs:
            consumers[p] = consumers.get(p, 0) + 1
    views = {}
    for G in reversed(groups):
        c = G.sink
        n = g.nodes[c]
        if n.op != "CONCAT":
            continue
        ax = int(n.attrs["axis"])
        outer = numel(n.shape[:ax])
        inner_c = numel(n.shape[ax:])
        if c in views:
            root, o_r, inner_root, base, _ = views[c]
            if o_r != outer:
                continue
        else:
            root, inner_root, base = c, inner_c, 0
        off = 0
        for v in n.preds:
            inner_v = numel(g.nodes[v].shape[ax:])
            nv = g.nodes[v]
            if (v in sink_of and nv.op not in LEAF and nv.op not in NO_VIEW_PRODUCERS and v not in keep
                    and consumers.get(v, 0) == 1 and n.preds.count(v) == 1):
                views[v] = (root, outer, inner_root, base + off, inner_v)
            off += inner_v
    return views


def plan_memory(g, groups, keep, flags):
    """Algorithm 1 over groups in Gamma order (SURVEY §8(c) c7-algo + R13 + R14)."""
    X = set()
    for G in groups:
        for p in G.inputs:
            if g.nodes[p].op in LEAF:
                X.add(p)
    refs = {}
    for G in groups:
        for p in G.inputs:
            if p not in X:
                refs[p] = refs.get(p, 0) + 1
    plan = Plan()
    plan.views = views = concat_views(g, groups, keep, flags)
    reusable = set()
    size = plan.size
    incremental = bool(flags & FLAG_INCREMENTAL)

    for G in groups:
        released = []

        def release(ps):
            for p in ps:
                refs[p] -= 1
                if refs[p] == 0 and p not in keep and p not in views:
                    reusable.add(plan.block[p])
                    released.append(p)

        pool_inputs = [p for p in G.inputs if p not in X]
        dn = dom_numel(g, G)
        if G.safe:
            release([p for p in pool_inputs if numel(g.nodes[p].shape) == dn])
        for m in G.materialised:
            nb = 4 * numel(g.nodes[m].shape)
            if m in views or m in plan.block:  # R14: the family's root block
                root = views[m][0] if m in views else m
                if root not in plan.block:
                    plan.block[root], _ = find_best_block(reusable, size, 4 * numel(g.nodes[root].shape))
                plan.block[m] = plan.block[root]
            elif incremental and m in keep:
                size.append(nb)
                plan.block[m] = len(size) - 1
            else:
                nm = numel(g.nodes[m].shape)
                pref = {plan.block[p] for p in released
                        if numel(g.nodes[p].shape) == nm and plan.block[p] in reusable}
                plan.block[m], _ = find_best_block(reusable, size, nb, pref)
        if G.safe:
            release([p for p in pool_inputs if numel(g.nodes[p].shape) != dn])
        else:
            release(pool_inputs)

    off = 0
    for s in size:
        plan.offsets.append(off)
        off += align_up(s)
    plan.pool_bytes = off
    plan.plan_bytes = sum(size)
    return plan
