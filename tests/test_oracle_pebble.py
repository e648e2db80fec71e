"""Pebble-game oracle (Definition 3) pinned to the
paper's printed values (Figs. 2 and 3) and to an independent brute force, and
the planner's space certified against it on the uniform-size examples."""
import random

from oracle.dump import compile_graph
from oracle.graph import Graph
from oracle.pebble import (brute_force_min_time, min_time, pareto_frontier, plan_pebbles, replay,
                           time_minimal_space)
from oracle.schedule import FLAG_NO_FUSION

# Fig. 1 / Fig. 2 (easypebbling): 0 = Const 2, 1 = x1, 2 = x2, 3 = x3, 4 = x4, 5 = x5
FIG1 = (6, [(0, 2), (1, 2), (2, 4), (3, 4), (4, 5)], [5])
# Fig. 3 (hardpebbling, edge list P:181)
FIG3 = (6, [(0, 1), (1, 5), (1, 2), (2, 4), (3, 4), (4, 5)], [5])


def test_fig2_space2_time6_optimal():
    """the Fig. 1 graph pebbles with space 2 and time 6, both minimal."""
    assert min_time(*FIG1, k=1) is None
    assert min_time(*FIG1, k=2) == 6
    assert pareto_frontier(*FIG1) == [(2, 6)]


def test_fig3_tradeoff():
    """time 6 with space 3, or time 8 with space 2; never both (2, 6)."""
    assert min_time(*FIG3, k=3) == 6
    assert min_time(*FIG3, k=2) == 8
    front = pareto_frontier(*FIG3)
    assert (3, 6) in front and (2, 8) in front and (2, 6) not in front


def test_strategies_replay_legally():
    for dag, k in ((FIG1, 2), (FIG3, 2), (FIG3, 3)):
        t, moves = min_time(*dag, k=k, with_strategy=True)
        space, time = replay(*dag, moves)
        assert time == t and space <= k


def test_chain_slides_with_one_pebble():
    """A path graph is pebbled by one pebble sliding along it: (1, n)."""
    n = 5
    assert pareto_frontier(n, [(i, i + 1) for i in range(n - 1)], [n - 1]) == [(1, n)]


def _random_dag(rng, n):
    edges = [(a, b) for b in range(1, n) for a in range(b) if rng.random() < 0.35]
    sinks = [v for v in range(n) if not any(a == v for a, _ in edges)]
    return n, edges, sinks[:2]


def test_search_equals_brute_force_on_small_dags():
    rng = random.Random(1812)
    for _ in range(40):
        n, edges, outs = _random_dag(rng, rng.randint(2, 6))
        for k in range(1, n + 1):
            want = brute_force_min_time(n, edges, outs, k, max_time=2 * n + 2)
            got = min_time(n, edges, outs, k, time_cap=2 * n + 2)
            assert got == want, (n, edges, outs, k)


def test_more_pebbles_never_cost_time():
    rng = random.Random(7)
    for _ in range(30):
        n, edges, outs = _random_dag(rng, rng.randint(2, 7))
        ts = [min_time(n, edges, outs, k) for k in range(1, n + 1)]
        ts = [t for t in ts if t is not None]
        assert all(a >= b for a, b in zip(ts, ts[1:]))


def _fig_graph(n, edges, inputs):
    g = Graph()
    ids = {}
    for v in range(n):
        ps = [a for a, b in edges if b == v]
        if not ps:
            ids[v] = g.add_leaf("VAR", (16,))
        elif len(ps) == 1:
            ids[v] = g.add_node("NEG", [ids[ps[0]]], {})
        else:
            ids[v] = g.add_node("ADD", [ids[p] for p in ps], {})
    return g, ids


def test_certify_planner_space():
    """certify_plan_space (SPEC mapping, stated in plan_pebbles): the node-level
    Alg. 1 plan never beats the exact optimum among time-minimal strategies."""
    for (n, edges, outs) in (FIG1, FIG3, (5, [(i, i + 1) for i in range(4)], [4])):
        g, ids = _fig_graph(n, edges, None)
        c = compile_graph(g, [ids[o] for o in outs], FLAG_NO_FUSION, do_optimise=False, compute_values=False)
        externals = [ids[v] for v in range(n) if g.nodes[ids[v]].op == "VAR"]
        used = plan_pebbles(c.plan.block, externals)
        best = time_minimal_space(n, edges, outs)
        assert used >= best
        assert time_minimal_space(*FIG3) == 3 and time_minimal_space(*FIG1) == 2
