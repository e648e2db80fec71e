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
"""
from __future__ import annotations

from .ops import LEAF, numel
from .schedule import FLAG_INCREMENTAL, dom_numel

ALIGN = 256


def align_up(x, a=ALIGN):
    return (x + a - 1) // a * a


class Plan:
    def __init__(self):
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


def plan_memory(g, groups, keep, flags):
    """Algorithm 1 over groups in Gamma order (SURVEY §8(c) c7-algo + R13)."""
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
    reusable = set()
    size = plan.size
    incremental = bool(flags & FLAG_INCREMENTAL)

    for G in groups:
        released = []

        def release(ps):
            for p in ps:
                refs[p] -= 1
                if refs[p] == 0 and p not in keep:
                    reusable.add(plan.block[p])
                    released.append(p)

        pool_inputs = [p for p in G.inputs if p not in X]
        dn = dom_numel(g, G)
        if G.safe:
            release([p for p in pool_inputs if numel(g.nodes[p].shape) == dn])
        for m in G.materialised:
            nb = 4 * numel(g.nodes[m].shape)
            if incremental and m in keep:
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
