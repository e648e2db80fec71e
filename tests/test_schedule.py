"""Executor order with batched collectives (csrc/schedule.cpp), CPU only.

The property that makes a reordering safe is fixed by the memory model, not by
the scheduler: two groups may swap only if neither writes a pool block the
other reads or writes (Alg. 1 reuses blocks) and they do not share
the workspace.  These tests check that property by brute force over every pair,
on random access sets and on the data-parallel C3 / C4 plans of the ORACLE's
planner (one AllReduce per gradient), where the
collectives must also come out batched.
"""
import random

import pytest

from oracle.dump import compile_graph
from oracle.graph import from_spec
from paper_1812_03770_b200 import cg
from paper_1812_03770_b200.dist import dp_spec
from workloads import configs


def _conflict(a, b, rd, wr, ws):
    return bool(set(wr[a]) & set(rd[b]) or set(rd[a]) & set(wr[b]) or set(wr[a]) & set(wr[b]) or (ws[a] and ws[b]))


def _check_valid(steps, rd, wr, ws, coll, active=None):
    ng = len(rd)
    act = [True] * ng if active is None else [bool(x) for x in active]
    order = [gi for s in steps for gi in s]
    assert sorted(order) == [gi for gi in range(ng) if act[gi]], "not a permutation of the active groups"
    pos = {gi: k for k, s in enumerate(steps) for gi in s}
    for s in steps:
        if len(s) > 1:
            assert all(coll[gi] for gi in s), "only collectives share a step"
            for i in range(len(s)):
                for j in range(i + 1, len(s)):
                    assert not _conflict(s[i], s[j], rd, wr, ws), "conflicting collectives batched"
    for a in order:
        for b in order:
            if a < b and _conflict(a, b, rd, wr, ws):
                assert pos[a] < pos[b], f"conflicting groups {a} < {b} reordered"


@pytest.mark.parametrize("seed", range(300))
def test_random_access_sets(seed):
    rng = random.Random(seed)
    ng = rng.randint(1, 40)
    nb = rng.randint(1, 12)
    rd = [rng.sample(range(nb), rng.randint(0, min(3, nb))) for _ in range(ng)]
    wr = [rng.sample(range(nb), rng.randint(0, min(2, nb))) for _ in range(ng)]
    ws = [rng.random() < 0.15 for _ in range(ng)]
    coll = [rng.random() < 0.3 for _ in range(ng)]
    active = [rng.random() < 0.85 for _ in range(ng)] if seed % 3 == 0 else None
    steps = cg.collective_schedule(rd, wr, ws, coll, active)
    _check_valid(steps, rd, wr, ws, coll, active)


def test_no_collectives_is_gamma_order():
    rd = [[0], [1], [0, 1], []]
    wr = [[1], [2], [0], [3]]
    steps = cg.collective_schedule(rd, wr, [0] * 4, [0] * 4)
    assert steps == [[0], [1], [2], [3]]


def test_independent_collectives_batch():
    # g0, g1 produce gradients (blocks 0, 1); AR g2, g4 in place; SGD g3, g5 read them
    rd = [[], [], [0], [0], [1], [1]]
    wr = [[0], [1], [0], [2], [1], [3]]
    coll = [0, 0, 1, 0, 1, 0]
    steps = cg.collective_schedule(rd, wr, [0] * 6, coll)
    assert steps == [[0], [1], [2, 4], [3], [5]]
    # a later group that overwrites the first gradient's block forces the flush before it
    rd2 = rd + [[]]
    wr2 = wr + [[0]]
    steps = cg.collective_schedule(rd2, wr2, [0] * 7, coll + [0])
    _check_valid(steps, rd2, wr2, [0] * 7, coll + [0])
    assert steps.index([6]) > [gi for s in steps for gi in s].index(3)


def _oracle_access_sets(spec):
    og, oo = from_spec(spec)
    c = compile_graph(og, oo, 0, compute_values=False)
    G = c.opt.g
    blk = c.plan.block
    rd, wr, coll = [], [], []
    for gr in c.groups:
        rd.append(sorted({blk[p] for p in gr.inputs if p in blk}))
        wr.append(sorted({blk[m] for m in gr.materialised if m in blk}))
        coll.append(G.nodes[gr.sink].op == "ALLREDUCE_SUM")
    ws = [G.nodes[gr.sink].op in ("DOT", "CONV2D", "CONV2D_BWD_INPUT", "CONV2D_BWD_KERNEL") or gr.kind == "red"
          for gr in c.groups]
    return rd, wr, ws, coll


@pytest.mark.parametrize("fn,batch,n_ar,max_batches", [(configs.c3, 4096, 6, 2), (configs.c4, 8192, 10, 3)])
def test_dp_training_plans_batch_allreduces(fn, batch, n_ar, max_batches):
    """On the planner's own C3 / C4 plans (dp2 rank 0) the reordering is valid and
    the per-gradient AllReduces come out in a few batches instead of n_ar calls."""
    rd, wr, ws, coll = _oracle_access_sets(dp_spec(fn, batch, 0, 2))
    assert sum(coll) == n_ar
    steps = cg.collective_schedule(rd, wr, ws, coll)
    _check_valid(steps, rd, wr, ws, coll)
    coll_steps = [s for s in steps if coll[s[0]]]
    print(fn.__name__, "collective steps:", [len(s) for s in coll_steps])
    assert len(coll_steps) <= max_batches
