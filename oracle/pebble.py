"""Exact pebble game (Definition 3) on small DAGs — ORACLE, test
infrastructure only.

Moves: (1) place a pebble on a vertex with no predecessor; (2) if all
predecessors of v are pebbled, place a pebble on v or *slide* one from a
predecessor to v; (3) remove any pebble.  Space = maximum number of pebbles in
use; time = number of placements (slides count, removals do not).  Goal:
every output vertex pebbled at least once.

``min_time`` is a 0-1 breadth-first search over states (pebbled set, outputs
reached) with at most ``k`` pebbles: placements cost 1, removals cost 0.  It is
exponential in |V| (the general problem is PSPACE-complete), so it is
restricted to |V| <= 20.  ``brute_force_min_time`` is an independent naive
iterative-deepening enumeration of move sequences used only to pin the search.
"""
from __future__ import annotations

from collections import deque

MAX_V = 20


def _preds(n, edges):
    p = [set() for _ in range(n)]
    for a, b in edges:
        p[b].add(a)
    return p


def _moves(state, preds, k):
    """(move, new_state, cost) for every legal move from ``state`` (a frozenset)."""
    n = len(preds)
    out = []
    for v in state:  # (3) remove
        out.append((("remove", v), state - {v}, 0))
    for v in range(n):
        if v in state:
            continue
        if preds[v] and not preds[v] <= state:
            continue
        if len(state) < k:  # (1)/(2) place
            out.append((("place", v), state | {v}, 1))
        for u in preds[v]:  # (2) slide from a predecessor
            out.append((("slide", u, v), (state - {u}) | {v}, 1))
    return out


def min_time(n: int, edges, outputs, k: int, time_cap: int | None = None, with_strategy: bool = False):
    """Minimal time of a strategy with space <= k pebbling every output once, or
    None if there is none within ``time_cap`` (default 4|V|)."""
    if n > MAX_V:
        raise ValueError(f"exact pebbling limited to {MAX_V} vertices")
    preds = _preds(n, edges)
    outs = frozenset(outputs)
    cap = 4 * n if time_cap is None else time_cap
    start = (frozenset(), frozenset())
    dist = {start: 0}
    parent = {start: None}
    dq = deque([start])
    while dq:
        st = dq.popleft()
        t = dist[st]
        peb, reached = st
        if reached == outs:
            if not with_strategy:
                return t
            moves = []
            while parent[st] is not None:
                prev, mv = parent[st]
                moves.append(mv)
                st = prev
            return t, moves[::-1]
        for mv, nxt, cost in _moves(peb, preds, k):
            nt = t + cost
            if nt > cap:
                continue
            ns = (nxt, reached | (nxt & outs))
            if ns not in dist or nt < dist[ns]:
                dist[ns] = nt
                parent[ns] = (st, mv)
                if cost == 0:
                    dq.appendleft(ns)
                else:
                    dq.append(ns)
    return None


def pareto_frontier(n: int, edges, outputs, time_cap: int | None = None):
    """Non-dominated (space, time) pairs ("cannot reach the minimal values of both")."""
    pts = []
    best = None
    for k in range(1, n + 1):
        t = min_time(n, edges, outputs, k, time_cap)
        if t is None:
            continue
        if best is None or t < best:
            pts.append((k, t))
            best = t
    return pts


def replay(n: int, edges, outputs, moves):
    """Independent rule checker (Definition 3): returns (space, time) of a legal
    strategy reaching the goal, raises ValueError otherwise."""
    preds = _preds(n, edges)
    peb, seen = set(), set()
    space = time = 0
    for mv in moves:
        if mv[0] == "remove":
            if mv[1] not in peb:
                raise ValueError(f"remove of unpebbled {mv[1]}")
            peb.discard(mv[1])
            continue
        v = mv[-1]
        if v in peb or not preds[v] <= peb:
            raise ValueError(f"illegal move {mv}")
        if mv[0] == "slide":
            if mv[1] not in preds[v]:
                raise ValueError(f"slide from a non-predecessor {mv}")
            peb.discard(mv[1])
        peb.add(v)
        seen.add(v)
        time += 1
        space = max(space, len(peb))
    if not set(outputs) <= seen:
        raise ValueError("outputs not all pebbled")
    return space, time


def brute_force_min_time(n: int, edges, outputs, k: int, max_time: int):
    """Naive iterative deepening over move sequences (no memoisation of costs),
    for DAGs of a handful of vertices: the pin of ``min_time``."""
    preds = _preds(n, edges)
    outs = set(outputs)

    def dfs(peb, seen, budget, depth, visited):
        if outs <= seen:
            return True
        if depth > 3 * n + max_time:
            return False
        key = (frozenset(peb), frozenset(seen & outs), budget)
        if key in visited:
            return False
        visited.add(key)
        for v in list(peb):
            if dfs(peb - {v}, seen, budget, depth + 1, visited):
                return True
        if budget == 0:
            return False
        for v in range(n):
            if v in peb or not preds[v] <= peb:
                continue
            if len(peb) < k and dfs(peb | {v}, seen | {v}, budget - 1, depth + 1, visited):
                return True
            for u in preds[v]:
                if dfs((peb - {u}) | {v}, seen | {v}, budget - 1, depth + 1, visited):
                    return True
        return False

    for t in range(0, max_time + 1):
        if dfs(frozenset(), set(), t, 0, set()):
            return t
    return None


def plan_pebbles(block_of: dict, externals) -> int:
    """Pebble count implied by a node-level memory plan (certify_plan_space's
    mapping, stated explicitly): every external vertex (Var/Const) holds its own
    pebble for the whole evaluation (inputs are user-owned), and every
    pool block is one pebble (blocks are reused, never duplicated)."""
    return len(set(externals)) + len(set(block_of.values()))


def time_minimal_space(n: int, edges, outputs):
    """Smallest k whose minimal time equals the time-minimal |ancestors(outputs)|
    (every needed vertex pebbled exactly once)."""
    preds = _preds(n, edges)
    need, stack = set(), list(outputs)
    while stack:
        v = stack.pop()
        if v not in need:
            need.add(v)
            stack.extend(preds[v])
    for k in range(1, n + 1):
        if min_time(n, edges, outputs, k) == len(need):
            return k
    return None
