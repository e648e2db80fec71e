"""The paper's pattern rewrites (ORACLE — test infrastructure only).

"Some patterns of nodes can be fused ... an FMA (fused-multiply-add) node can
replace a multiplication followed by an addition to reduce memory access and
improve numerical accuracy.  A common subpattern of AdaGrad ... can also be
fused into one node" and "useless calculations, such as adding zero, dividing
by one, multiplying by zero or one, ... are automatically optimised".

Readings (SPEC S:195-230 for the concrete patterns):
* keep = outputs + update sources (raw ids); keep nodes are never removed, and
  never absorbed as an interior node of a fusion (an FMA/AdaGrad *root* may be
  a keep node: it keeps its id and changes its operation);
* "single consumer" = exactly one consuming edge among live nodes;
* identities (only user / rewritten Consts whose every element is exactly 0 or
  1, and only when the surviving operand already has the result's shape, so
  broadcasting never changes a shape): x+0, 0+x, x-0, x*1, 1*x, x/1 -> x
  (recorded in rep like a CSE merge); x*0, 0*x -> a Const of zeros (id kept);
  the paper's "repeating the input of an operation supporting broadcasting"
  has no counterpart: this op set has no Repeat;
* FusedAdagrad(g, s, lr, eps) = lr*g / (sqrt(s) + eps) replaces
  DIV(MUL(lr, g), ADD(SQRT(s), eps)) with scalar Consts lr, eps (either
  operand order); the three interior nodes must be single-consumer and not kept;
* FMA(a, b, c) replaces ADD(MUL(a, b), c) or ADD(c, MUL(a, b)) (left operand
  tried first) when the MUL is single-consumer and not kept;
* order: one ascending-id sweep each of identities, AdaGrad, FMA, repeated until
  a whole round changes nothing; then CSE -> CF -> DCE as before.
"""
from __future__ import annotations

import numpy as np

RW_IDENTITY, RW_FMA, RW_ADAGRAD = 1, 2, 4
RW_ALL = RW_IDENTITY | RW_FMA | RW_ADAGRAD


def _const_all(g, v, x):
    n = g.nodes[v]
    if n.op != "CONST":
        return False
    val = g.const_value(v)
    return bool(np.all(val == np.float32(x)))


def _scalar_const(g, v):
    n = g.nodes[v]
    return n.op == "CONST" and all(d == 1 for d in n.shape)


def rewrite(g, outputs, flags, dead: set):
    """Apply the rewrites in place on ``g`` (a clone).  Returns (rep, counts, lists)."""
    keep = set(outputs) | {u for u, _ in g.updates}
    rep = {}
    counts = {"rw_identity": 0, "rw_zeroed": 0, "rw_fma": 0, "rw_adagrad": 0}
    lists = {"identity": [], "zeroed": [], "fma": [], "adagrad": []}

    def res(v):
        while v in rep:
            v = rep[v]
        return v

    def redirect():
        for n in g.nodes:
            if n.id not in dead:
                n.preds = [res(p) for p in n.preds]

    def uses():
        u = {}
        for n in g.nodes:
            if n.id in dead:
                continue
            for p in n.preds:
                u[p] = u.get(p, 0) + 1
        return u

    def interior_ok(v, cnt):
        return v not in dead and v not in keep and cnt.get(v, 0) == 1

    while True:
        changed = False
        if flags & RW_IDENTITY:
            redirect()
            for n in g.nodes:
                v = n.id
                if v in dead or v in keep or n.op not in ("ADD", "SUB", "MUL", "DIV"):
                    continue
                n.preds = [res(p) for p in n.preds]
                a, b = n.preds
                sa, sb = g.nodes[a].shape, g.nodes[b].shape
                to = None
                if n.op == "ADD":
                    if _const_all(g, b, 0.0) and sa == n.shape:
                        to = a
                    elif _const_all(g, a, 0.0) and sb == n.shape:
                        to = b
                elif n.op == "SUB":
                    if _const_all(g, b, 0.0) and sa == n.shape:
                        to = a
                elif n.op == "MUL":
                    if _const_all(g, b, 1.0) and sa == n.shape:
                        to = a
                    elif _const_all(g, a, 1.0) and sb == n.shape:
                        to = b
                    elif _const_all(g, a, 0.0) or _const_all(g, b, 0.0):
                        n.op, n.preds, n.attrs, n.data = "CONST", [], {}, None
                        n.value = np.zeros(n.shape, np.float32)
                        counts["rw_zeroed"] += 1
                        lists["zeroed"].append(v)
                        changed = True
                        continue
                elif n.op == "DIV":
                    if _const_all(g, b, 1.0) and sa == n.shape:
                        to = a
                if to is not None:
                    rep[v] = to
                    dead.add(v)
                    counts["rw_identity"] += 1
                    lists["identity"].append(v)
                    changed = True
        if flags & RW_ADAGRAD:
            redirect()
            cnt = uses()
            for n in g.nodes:
                v = n.id
                if v in dead or n.op != "DIV":
                    continue
                num, den = n.preds
                N, D = g.nodes[num], g.nodes[den]
                if N.op != "MUL" or D.op != "ADD" or not interior_ok(num, cnt) or not interior_ok(den, cnt):
                    continue
                if _scalar_const(g, N.preds[0]):
                    lr, gg = N.preds[0], N.preds[1]
                elif _scalar_const(g, N.preds[1]):
                    lr, gg = N.preds[1], N.preds[0]
                else:
                    continue
                d0, d1 = D.preds
                if g.nodes[d0].op == "SQRT" and _scalar_const(g, d1):
                    q, eps = d0, d1
                elif g.nodes[d1].op == "SQRT" and _scalar_const(g, d0):
                    q, eps = d1, d0
                else:
                    continue
                if not interior_ok(q, cnt):
                    continue
                s = g.nodes[q].preds[0]
                n.op, n.preds = "FUSED_ADAGRAD", [gg, s, lr, eps]
                dead.update((num, den, q))
                counts["rw_adagrad"] += 1
                lists["adagrad"].append(v)
                changed = True
        if flags & RW_FMA:
            redirect()
            cnt = uses()
            for n in g.nodes:
                v = n.id
                if v in dead or n.op != "ADD":
                    continue
                for side in (0, 1):
                    m, c = n.preds[side], n.preds[1 - side]
                    if g.nodes[m].op == "MUL" and interior_ok(m, cnt):
                        a, b = g.nodes[m].preds
                        n.op, n.preds = "FMA", [a, b, c]
                        dead.add(m)
                        counts["rw_fma"] += 1
                        lists["fma"].append(v)
                        changed = True
                        break
        if not changed:
            break
    redirect()
    return rep, counts, lists
