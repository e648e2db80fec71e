"""Property pins of the oracle on seeded random DAGs and small training graphs (CPU only).

- planner soundness: brute-force liveness on every plan, pool <= unshared
- Gamma is topological (Def. 2); groups are convex
- incremental engine (c9) run on SIMULATED BLOCKS equals fresh eager evaluation
  after every assign/eval step — the brute-force pin of both the
  plan and the recompute-set rules
- Fig. 1 incremental invariant: changing x3 does not recompute x2
- the hand-written backward graphs of C3/C4 match f64 finite differences
"""
import random

import numpy as np
import pytest

from oracle.dump import compile_graph
from oracle.eager import ancestors, evaluate, leaf_values
from oracle.graph import from_spec
from oracle.incremental import EVAL_NO_UPDATE, BlockSim, IncrementalModel
from oracle.ops import EW
from oracle.schedule import FLAG_INCREMENTAL, FLAG_NO_FUSION
from oracle.validate import validate_plan
from tests.randgraph import random_spec
from workloads import configs

MODES = [0, FLAG_NO_FUSION, FLAG_INCREMENTAL, FLAG_INCREMENTAL | FLAG_NO_FUSION]


@pytest.mark.parametrize("mode", MODES)
def test_random_plans_valid(mode):
    for seed in range(250):
        g, outs = from_spec(random_spec(seed))
        c = compile_graph(g, outs, mode, compute_values=False)
        assert validate_plan(c) == [], seed
        assert c.plan.plan_bytes <= c.unshared_bytes or not c.groups
        rank = c.rank
        for n in c.gamma:
            for p in c.g.nodes[n].preds:
                assert rank[p] < rank[n]
        sinks = [G.sink for G in c.groups]
        assert [rank[s] for s in sinks] == sorted(rank[s] for s in sinks)
        for G in c.groups:
            mem = set(G.members)
            for m in G.members:
                if m == G.sink:
                    continue
                cons = [v for v in c.gamma if m in c.g.nodes[v].preds]
                assert all(v in mem for v in cons), (seed, "convexity")
            ops = {c.g.nodes[m].op for m in G.members}
            if len(G.members) > 1:
                assert ops <= EW | {"SUM", "MAX"}
                assert all(c.g.nodes[m].op in EW for m in G.members if m != G.sink)


@pytest.mark.parametrize("mode", MODES)
def test_incremental_block_simulation_equals_eager(mode):
    for seed in range(120):
        spec = random_spec(seed, simple_values=True)
        g, outs = from_spec(spec)
        c = compile_graph(g, outs, mode)
        rng = random.Random(seed * 7 + mode)
        # oracle's reference: fresh eager evaluation of the OPTIMISED graph (bit-identical
        # to the raw graph's: CSE/CF do the same per-node arithmetic)
        state = leaf_values(c.g)
        sim = BlockSim(c, state)
        vars_ = [v for v in c.gamma if c.g.nodes[v].op == "VAR"]
        for step in range(8):
            if vars_ and rng.random() < 0.7:
                x = rng.choice(vars_)
                val = np.float32(rng.uniform(0.5, 1.5)) * np.ones(c.g.nodes[x].shape, np.float32)
                state[x] = val
                sim.assign(x, val)
            full = rng.random() < 0.6
            ev = c.outputs if full else rng.sample(c.outputs, 1)
            flags = 0 if rng.random() < 0.7 else EVAL_NO_UPDATE
            got, R = sim.eval(ev, flags)
            ref = evaluate(c.g, state, ancestors(c.g, list(ev) + [u for u, _ in c.g.updates]))
            for o in ev:
                assert np.array_equal(got[o], ref[o], equal_nan=True), (seed, mode, step, o)
            if not flags & EVAL_NO_UPDATE:
                for u, v in c.g.updates:
                    state[v] = ref[u].copy()


def test_fig1_incremental_invariant():
    g, outs = from_spec(configs.c1(16))
    for mode, x2_recomputed in [(FLAG_INCREMENTAL, False), (0, True), (FLAG_NO_FUSION, True)]:
        c = compile_graph(g, outs, mode)
        m = IncrementalModel(c)
        m.eval(outs)
        assert all(m.count[v] == 1 for v in (2, 4, 5))
        m.assign(3)  # change x3 only
        R = m.eval(outs)
        assert m.count[4] == 2 and m.count[5] == 2
        assert (m.count[2] == 2) == x2_recomputed, mode
        if mode == FLAG_INCREMENTAL:
            assert [c.groups[i].members for i in sorted(R)] == [[4, 5]]
        m.eval(outs)  # nothing changed: nothing recomputed
        assert m.count[5] == 2


def _grad_of(g, update_source):
    """Walk Wn = SUB(W, MUL(ALLREDUCE_SUM(grad), lr)) back to the raw gradient node."""
    sub = g.nodes[update_source]
    mul = g.nodes[sub.preds[1]]
    ar = g.nodes[mul.preds[0]]
    return ar.preds[0] if ar.op == "ALLREDUCE_SUM" else mul.preds[0]


@pytest.mark.parametrize("which", ["C3", "C4"])
def test_backward_graphs_finite_differences(which):
    if which == "C3":
        spec = configs.c3(batch=4, widths=(6, 5, 4, 3))
    else:
        spec = configs.c4(batch=2, hw=12)
    g, outs = from_spec(spec)
    loss = outs[0]
    rng = np.random.default_rng(5)
    base = {k: v.astype(np.float64) for k, v in leaf_values(g).items()}
    for v in g.var_ids():
        if g.nodes[v].name.startswith("b"):
            base[v] = rng.uniform(-0.1, 0.1, g.nodes[v].shape)  # nonzero biases

    def run(vals):
        return evaluate(g, vals, dtype=np.float64)

    ref = run(base)
    checked = 0
    for u, v in g.updates:
        grad = ref[_grad_of(g, u)]
        flat = base[v].ravel()
        for _ in range(4):
            k = rng.integers(flat.size)
            for attempt in range(5):
                eps = 1e-6
                plus, minus = dict(base), dict(base)
                p = flat.copy(); p[k] += eps
                m = flat.copy(); m[k] -= eps
                plus[v] = p.reshape(base[v].shape)
                minus[v] = m.reshape(base[v].shape)
                rp, rm = run(plus), run(minus)
                # kinks (ReLU / max-pool ties) crossing -> resample
                masks_equal = all(
                    np.array_equal(rp[n.id] > 0, rm[n.id] > 0)
                    for n in g.nodes if n.op in ("RELU", "MAXPOOL2D"))
                if masks_equal:
                    break
                k = rng.integers(flat.size)
            fd = (float(rp[loss].ravel()[0]) - float(rm[loss].ravel()[0])) / (2 * eps)
            an = float(grad.ravel()[k])
            assert abs(fd - an) <= 1e-6 + 1e-4 * abs(an), (which, g.nodes[v].name, k, fd, an)
            checked += 1
    assert checked >= 4 * len(g.updates)
