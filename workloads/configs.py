"""Graph specs of the BASELINE.json configs C1-C5.

A graph spec is plain data: a list of node records in creation order plus the
declared outputs and update edges.  It is the *workload*, consumed by both the
oracle (oracle/graph.py) and the CUDA path's Python binding
(paper_1812_03770_b200/cg.py), each with its own parser.  This module holds
none of the method's arithmetic: no shape inference, no rewriting, no
planning, no evaluation.  Shapes appear only where a leaf needs one (Var,
Const) or where an op's attribute is a shape (RESHAPE dims, conv-backward
input sizes).

Node record:  {"id": i, "op": "MUL", "preds": [..], "attrs": {..}}
Leaf record:  {"id": i, "op": "VAR"|"CONST", "preds": [], "attrs": {},
               "name": s, "shape": [..], "data": <workloads.gen data spec>}
"""
from __future__ import annotations

import math


class Spec:
    """Records a program as a graph spec, in creation order."""

    def __init__(self, name: str, **meta):
        self.name = name
        self.nodes: list[dict] = []
        self.outputs: list[int] = []
        self.updates: list[list[int]] = []
        self.meta = dict(meta)

    # leaves -----------------------------------------------------------
    def _leaf(self, op, name, shape, data):
        i = len(self.nodes)
        self.nodes.append({"id": i, "op": op, "preds": [], "attrs": {}, "name": name,
                           "shape": [int(d) for d in shape], "data": data})
        return i

    def var(self, name, shape, data=None):
        return self._leaf("VAR", name, shape, data or {"kind": "zeros"})

    def const(self, name, shape, data):
        return self._leaf("CONST", name, shape, data)

    def scalar(self, name, value):
        return self._leaf("CONST", name, [], {"kind": "literal", "values": [float(value)]})

    # ops --------------------------------------------------------------
    def op(self, op, *preds, **attrs):
        i = len(self.nodes)
        self.nodes.append({"id": i, "op": op, "preds": [int(p) for p in preds], "attrs": dict(attrs)})
        return i

    def output(self, *ids):
        self.outputs.extend(int(i) for i in ids)

    def update(self, u, var):
        self.updates.append([int(u), int(var)])

    def to_dict(self):
        return {"name": self.name, "nodes": self.nodes, "outputs": list(self.outputs),
                "updates": [list(p) for p in self.updates], "meta": dict(self.meta)}

    def shape_of(self, i):
        """Shape of a leaf (accumulators copy their parameter's shape)."""
        return list(self.nodes[i]["shape"])

    def leaf_ids(self, op=None):
        return [n["id"] for n in self.nodes if n["op"] in ("VAR", "CONST") and (op is None or n["op"] == op)]


def U(tag, lo, hi):
    return {"kind": "uniform", "tag": tag, "lo": float(lo), "hi": float(hi)}


def glorot(tag, fan_in, fan_out):
    a = math.sqrt(6.0 / (fan_in + fan_out))
    return U(tag, -a, a)


def he(tag, fan_in):
    a = math.sqrt(6.0 / fan_in)
    return U(tag, -a, a)


ZEROS = {"kind": "zeros"}

# ---------------------------------------------------------------------------
# C1: Figure 1
# ---------------------------------------------------------------------------


def c1(n: int = 1024) -> dict:
    """x2 <- 2 - x1; x4 <- x2 * x3; x5 <- sin x4.  Ids 0..5 = Fig. 2 labels."""
    s = Spec("C1", n=n)
    c = s.scalar("two", 2.0)
    x1 = s.var("x1", [n], U("x1", 0.0, 4.0))
    x2 = s.op("SUB", c, x1)
    x3 = s.var("x3", [n], U("x3", -math.pi / 2, math.pi / 2))
    x4 = s.op("MUL", x2, x3)
    x5 = s.op("SIN", x4)
    s.output(x5)
    s.meta["reassign"] = {"x3": U("x3#2", -math.pi / 2, math.pi / 2)}
    return s.to_dict()


# ---------------------------------------------------------------------------
# C2: the 20-op elementwise/broadcast chain
# ---------------------------------------------------------------------------

C2_ROWS = 1 << 18
C2_COLS = 1024


def c2(rows: int = C2_ROWS, cols: int = C2_COLS) -> dict:
    s = Spec("C2", rows=rows, cols=cols)
    x = s.var("x", [rows, cols], U("x", -1, 1))
    y = s.var("y", [rows, cols], U("y", -1, 1))
    r = s.const("r", [1, cols], U("r", 0.5, 1.5))
    sh = s.const("s", [1, cols], U("s", -0.25, 0.25))
    c = s.const("c", [rows, 1], U("c", 0, 1))
    ka = s.scalar("ka", 0.5)
    kb = s.scalar("kb", 2.0)
    kc = s.scalar("kc", 0.044715)
    kd = s.scalar("kd", 0.7978845608)
    n1 = s.op("MUL", ka, kb)
    n2 = s.op("MUL", kc, n1)
    d = s.op("SUB", x, y)
    u = s.op("MUL", d, r)
    v = s.op("ADD", u, sh)
    v2 = s.op("MUL", v, v)
    v3 = s.op("MUL", v2, v)
    w = s.op("MUL", v3, n2)
    p = s.op("ADD", v, w)
    q = s.op("MUL", p, kd)
    th = s.op("TANH", q)
    e = s.op("ADD", th, n1)
    g = s.op("MUL", v, e)
    g2 = s.op("MUL", g, ka)
    v2b = s.op("MUL", v, v)
    m = s.op("MUL", v2b, c)
    nm = s.op("NEG", m)
    ex = s.op("EXP", nm)
    o = s.op("MUL", g2, ex)
    out = s.op("ADD", o, d)
    s.output(out)
    return s.to_dict()


C2_ALGO_BYTES_PER_ELEMENT_NOTE = "x, y read + out written = 12 B/element, plus c (4 B/row) and r, s (8 B/column)"


def c2_algo_bytes(rows: int = C2_ROWS, cols: int = C2_COLS) -> int:
    """Algorithmic HBM bytes of one C2 eval: x,y read, out written, c, r, s read once."""
    return 4 * (3 * rows * cols + rows + 2 * cols)


# ---------------------------------------------------------------------------
# Softmax cross-entropy (composition of MAX, SUB, EXP, SUM, LOG, MUL; §8(c) c1-defs)
# ---------------------------------------------------------------------------


def _softmax_xent(s: Spec, L, Y, batch_global: int):
    M = s.op("MAX", L, a0=1, a1=2)
    S = s.op("SUB", L, M)
    E = s.op("EXP", S)
    Ssum = s.op("SUM", E, a0=1, a1=2)
    P = s.op("DIV", E, Ssum)
    LS = s.op("LOG", Ssum)
    LP = s.op("SUB", S, LS)
    YL = s.op("MUL", Y, LP)
    T = s.op("SUM", YL, a0=0, a1=2)
    kneg = s.scalar("neg_inv_batch", -1.0 / batch_global)
    loss = s.op("MUL", T, kneg)
    D = s.op("SUB", P, Y)
    kinv = s.scalar("inv_batch", 1.0 / batch_global)
    dL = s.op("MUL", D, kinv)
    return loss, P, dL


def _adagrad(s: Spec, params_and_grads, lr: float, allreduce: bool, eps: float = 1e-8):
    """AdaGrad [adagrad]: s <- s + g*g; W <- W - lr*g / (sqrt(s) + eps), with an
    accumulator Var per parameter and two update edges per parameter.  The
    adjusted-gradient subgraph is the pattern the paper fuses into
    Fused_Adagrad."""
    klr = s.scalar("lr", lr)
    keps = s.scalar("eps", eps)
    for W, g in params_and_grads:
        if allreduce:
            g = s.op("ALLREDUCE_SUM", g)
        acc = s.var(f"acc_{s.nodes[W]['name']}", s.shape_of(W), ZEROS)
        acc_new = s.op("ADD", acc, s.op("MUL", g, g))
        step = s.op("DIV", s.op("MUL", klr, g), s.op("ADD", s.op("SQRT", acc_new), keps))
        s.update(s.op("SUB", W, step), W)
        s.update(acc_new, acc)


def _sgd(s: Spec, params_and_grads, lr: float, allreduce: bool):
    klr = s.scalar("lr", lr)
    for W, g in params_and_grads:
        if allreduce:
            g = s.op("ALLREDUCE_SUM", g)
        step = s.op("MUL", g, klr)
        Wn = s.op("SUB", W, step)
        s.update(Wn, W)


# ---------------------------------------------------------------------------
# C3: MNIST-shaped MLP 784-1024-1024-10, batch 4096, SGD with update edges
# ---------------------------------------------------------------------------


def c3(batch: int = 4096, widths=(784, 1024, 1024, 10), batch_global: int | None = None,
       lr: float = 0.05, allreduce: bool = True, optimizer: str = "sgd") -> dict:
    """Forward DOT->+b->RELU (x2), DOT->+b; softmax-xent; hand-written backward; SGD.

    ``batch`` is the local (per-rank) batch; ``batch_global`` scales the loss
    (1/B_global, §8(c) c10)."""
    bg = batch_global or batch
    s = Spec("C3", batch=batch, batch_global=bg, widths=list(widths), lr=lr)
    X = s.var("X", [batch, widths[0]], U("X", 0, 1))
    Y = s.var("Y", [batch, widths[-1]], {"kind": "onehot", "tag": "Y", "classes": widths[-1]})
    Ws, bs = [], []
    for li in range(len(widths) - 1):
        Ws.append(s.var(f"W{li + 1}", [widths[li], widths[li + 1]],
                        glorot(f"W{li + 1}", widths[li], widths[li + 1])))
        bs.append(s.var(f"b{li + 1}", [1, widths[li + 1]], ZEROS))
    h = X
    pre, acts = [], [X]
    nl = len(Ws)
    for li in range(nl):
        z = s.op("DOT", h, Ws[li], ta=0, tb=0)
        a = s.op("ADD", z, bs[li])
        pre.append(a)
        if li < nl - 1:
            h = s.op("RELU", a)
            acts.append(h)
        else:
            h = a
    L = h
    loss, P, dL = _softmax_xent(s, L, Y, bg)
    grads = [None] * nl
    d = dL
    for li in reversed(range(nl)):
        dW = s.op("DOT", acts[li], d, ta=1, tb=0)
        db = s.op("SUM", d, a0=0, a1=1)
        grads[li] = (dW, db)
        if li > 0:
            dh = s.op("DOT", d, Ws[li], ta=0, tb=1)
            d = s.op("RELU_GRAD", pre[li - 1], dh)
    pg = []
    for li in range(nl):
        pg.append((Ws[li], grads[li][0]))
        pg.append((bs[li], grads[li][1]))
    if optimizer == "adagrad":
        _adagrad(s, pg, lr, allreduce)
    else:
        _sgd(s, pg, lr, allreduce)
    s.output(loss, L)
    s.meta["per_iteration"] = ["X", "Y"]
    return s.to_dict()


# ---------------------------------------------------------------------------
# C4: LeNet-style CNN on 28x28x1, batch 8192
# ---------------------------------------------------------------------------


def c4(batch: int = 8192, batch_global: int | None = None, lr: float = 0.05, allreduce: bool = True,
       hw: int = 28) -> dict:
    bg = batch_global or batch
    s = Spec("C4", batch=batch, batch_global=bg, lr=lr, hw=hw)
    X = s.var("X", [batch, hw, hw, 1], U("X", 0, 1))
    Y = s.var("Y", [batch, 10], {"kind": "onehot", "tag": "Y", "classes": 10})
    W1 = s.var("W1", [5, 5, 1, 6], glorot("W1", 25 * 1, 25 * 6))
    b1 = s.var("b1", [1, 1, 1, 6], ZEROS)
    W2 = s.var("W2", [5, 5, 6, 16], glorot("W2", 25 * 6, 25 * 16))
    b2 = s.var("b2", [1, 1, 1, 16], ZEROS)
    h2w = (hw // 2 - 4) // 2
    flat = h2w * h2w * 16
    W3 = s.var("W3", [flat, 120], glorot("W3", flat, 120))
    b3 = s.var("b3", [1, 120], ZEROS)
    W4 = s.var("W4", [120, 84], glorot("W4", 120, 84))
    b4 = s.var("b4", [1, 84], ZEROS)
    W5 = s.var("W5", [84, 10], glorot("W5", 84, 10))
    b5 = s.var("b5", [1, 10], ZEROS)
    c1_ = s.op("CONV2D", X, W1, sh=1, sw=1, pad=1)
    a1 = s.op("ADD", c1_, b1)
    h1 = s.op("RELU", a1)
    p1 = s.op("MAXPOOL2D", h1, kh=2, kw=2, sh=2, sw=2, pad=0)
    c2_ = s.op("CONV2D", p1, W2, sh=1, sw=1, pad=0)
    a2 = s.op("ADD", c2_, b2)
    h2 = s.op("RELU", a2)
    p2 = s.op("MAXPOOL2D", h2, kh=2, kw=2, sh=2, sw=2, pad=0)
    f = s.op("RESHAPE", p2, dims=[batch, flat])
    z3 = s.op("DOT", f, W3, ta=0, tb=0)
    a3 = s.op("ADD", z3, b3)
    h3 = s.op("RELU", a3)
    z4 = s.op("DOT", h3, W4, ta=0, tb=0)
    a4 = s.op("ADD", z4, b4)
    h4 = s.op("RELU", a4)
    z5 = s.op("DOT", h4, W5, ta=0, tb=0)
    L = s.op("ADD", z5, b5)
    loss, P, dL = _softmax_xent(s, L, Y, bg)
    dW5 = s.op("DOT", h4, dL, ta=1, tb=0)
    db5 = s.op("SUM", dL, a0=0, a1=1)
    dh4 = s.op("DOT", dL, W5, ta=0, tb=1)
    da4 = s.op("RELU_GRAD", a4, dh4)
    dW4 = s.op("DOT", h3, da4, ta=1, tb=0)
    db4 = s.op("SUM", da4, a0=0, a1=1)
    dh3 = s.op("DOT", da4, W4, ta=0, tb=1)
    da3 = s.op("RELU_GRAD", a3, dh3)
    dW3 = s.op("DOT", f, da3, ta=1, tb=0)
    db3 = s.op("SUM", da3, a0=0, a1=1)
    df = s.op("DOT", da3, W3, ta=0, tb=1)
    dp2 = s.op("RESHAPE", df, dims=[batch, h2w, h2w, 16])
    dh2 = s.op("MAXPOOL2D_BWD", h2, dp2, kh=2, kw=2, sh=2, sw=2, pad=0)
    da2 = s.op("RELU_GRAD", a2, dh2)
    dW2 = s.op("CONV2D_BWD_KERNEL", p1, da2, sh=1, sw=1, pad=0, kh=5, kw=5)
    db2 = s.op("SUM", da2, a0=0, a1=3)
    dp1 = s.op("CONV2D_BWD_INPUT", da2, W2, sh=1, sw=1, pad=0, h=hw // 2, w=hw // 2)
    dh1 = s.op("MAXPOOL2D_BWD", h1, dp1, kh=2, kw=2, sh=2, sw=2, pad=0)
    da1 = s.op("RELU_GRAD", a1, dh1)
    dW1 = s.op("CONV2D_BWD_KERNEL", X, da1, sh=1, sw=1, pad=1, kh=5, kw=5)
    db1 = s.op("SUM", da1, a0=0, a1=3)
    _sgd(s, [(W1, dW1), (b1, db1), (W2, dW2), (b2, db2), (W3, dW3), (b3, db3),
             (W4, dW4), (b4, db4), (W5, dW5), (b5, db5)], lr, allreduce)
    s.output(loss, L)
    s.meta["per_iteration"] = ["X", "Y"]
    return s.to_dict()


# ---------------------------------------------------------------------------
# C5: InceptionV3-shaped inference graph
# ---------------------------------------------------------------------------


class _Inception:
    def __init__(self, s: Spec, batch: int):
        self.s = s
        self.batch = batch
        self.k = 0

    def cb(self, x, cin, cout, kh, kw, stride=1, pad=1):
        """CONV2D -> BN (SUB mean, DIV sqrt(var+eps), MUL gamma, ADD beta) -> RELU."""
        s = self.s
        self.k += 1
        k = self.k
        W = s.const(f"conv{k}.w", [kh, kw, cin, cout], he(f"conv{k}.w", kh * kw * cin))
        y = s.op("CONV2D", x, W, sh=stride, sw=stride, pad=pad)
        mean = s.const(f"bn{k}.mean", [cout], U(f"bn{k}.mean", -0.1, 0.1))
        var = s.const(f"bn{k}.var", [cout], U(f"bn{k}.var", 0.5, 1.5))
        eps = s.scalar(f"bn{k}.eps", 1e-3)
        beta = s.const(f"bn{k}.beta", [cout], U(f"bn{k}.beta", -0.1, 0.1))
        gamma = s.const(f"bn{k}.gamma", [cout], {"kind": "full", "value": 1.0})
        ve = s.op("ADD", var, eps)
        sd = s.op("SQRT", ve)
        t = s.op("SUB", y, mean)
        t = s.op("DIV", t, sd)
        t = s.op("MUL", t, gamma)
        t = s.op("ADD", t, beta)
        return s.op("RELU", t)

    def maxpool(self, x, k=3, stride=2, pad=0):
        return self.s.op("MAXPOOL2D", x, kh=k, kw=k, sh=stride, sw=stride, pad=pad)

    def avgpool(self, x, k=3, stride=1, pad=1):
        return self.s.op("AVGPOOL2D", x, kh=k, kw=k, sh=stride, sw=stride, pad=pad)

    def concat(self, *xs):
        return self.s.op("CONCAT", *xs, axis=3)


def c5(batch: int = 256, hw: int = 299, classes: int = 1000) -> dict:
    s = Spec("C5", batch=batch, hw=hw, classes=classes)
    net = _Inception(s, batch)
    X = s.var("X", [batch, hw, hw, 3], U("X", -1, 1))
    cb = net.cb
    x = cb(X, 3, 32, 3, 3, 2, 0)
    x = cb(x, 32, 32, 3, 3, 1, 0)
    x = cb(x, 32, 64, 3, 3)
    x = net.maxpool(x)
    x = cb(x, 64, 80, 1, 1, 1, 0)
    x = cb(x, 80, 192, 3, 3, 1, 0)
    x = net.maxpool(x)
    cin = 192
    for pool_w in (32, 64, 64):  # mixed0-2
        b1 = cb(x, cin, 64, 1, 1)
        b5 = cb(cb(x, cin, 48, 1, 1), 48, 64, 5, 5)
        b3 = cb(cb(cb(x, cin, 64, 1, 1), 64, 96, 3, 3), 96, 96, 3, 3)
        bp = cb(net.avgpool(x), cin, pool_w, 1, 1)
        x = net.concat(b1, b5, b3, bp)
        cin = 64 + 64 + 96 + pool_w
    # mixed3
    b3 = cb(x, cin, 384, 3, 3, 2, 0)
    bd = cb(cb(cb(x, cin, 64, 1, 1), 64, 96, 3, 3), 96, 96, 3, 3, 2, 0)
    bp = net.maxpool(x)
    x = net.concat(b3, bd, bp)
    cin = 384 + 96 + cin
    for c in (128, 160, 160, 192):  # mixed4-7
        b1 = cb(x, cin, 192, 1, 1)
        b7 = cb(cb(cb(x, cin, c, 1, 1), c, c, 1, 7), c, 192, 7, 1)
        bd = cb(x, cin, c, 1, 1)
        bd = cb(bd, c, c, 7, 1)
        bd = cb(bd, c, c, 1, 7)
        bd = cb(bd, c, c, 7, 1)
        bd = cb(bd, c, 192, 1, 7)
        bp = cb(net.avgpool(x), cin, 192, 1, 1)
        x = net.concat(b1, b7, bd, bp)
        cin = 768
    # mixed8
    b3 = cb(cb(x, cin, 192, 1, 1), 192, 320, 3, 3, 2, 0)
    b7 = cb(x, cin, 192, 1, 1)
    b7 = cb(b7, 192, 192, 1, 7)
    b7 = cb(b7, 192, 192, 7, 1)
    b7 = cb(b7, 192, 192, 3, 3, 2, 0)
    bp = net.maxpool(x)
    x = net.concat(b3, b7, bp)
    cin = 320 + 192 + cin
    for _ in range(2):  # mixed9-10
        b1 = cb(x, cin, 320, 1, 1)
        b3 = cb(x, cin, 384, 1, 1)
        b3 = net.concat(cb(b3, 384, 384, 1, 3), cb(b3, 384, 384, 3, 1))
        bd = cb(cb(x, cin, 448, 1, 1), 448, 384, 3, 3)
        bd = net.concat(cb(bd, 384, 384, 1, 3), cb(bd, 384, 384, 3, 1))
        bp = cb(net.avgpool(x), cin, 192, 1, 1)
        x = net.concat(b1, b3, bd, bp)
        cin = 320 + 768 + 768 + 192
    sp = (hw - 3) // 2 + 1 - 2          # stem convs: 149 -> 147 at 299
    sp = (sp - 3) // 2 + 1 - 2          # maxpool, 3x3 VALID conv: 73 -> 71
    sp = (sp - 3) // 2 + 1              # maxpool -> 35
    sp = (sp - 3) // 2 + 1              # mixed3 -> 17
    sp = (sp - 3) // 2 + 1  # mixed8 -> 8
    g = s.op("AVGPOOL2D", x, kh=sp, kw=sp, sh=sp, sw=sp, pad=0)
    f = s.op("RESHAPE", g, dims=[batch, cin])
    Wfc = s.const("fc.w", [cin, classes], glorot("fc.w", cin, classes))
    bfc = s.const("fc.b", [1, classes], U("fc.b", -0.1, 0.1))
    z = s.op("DOT", f, Wfc, ta=0, tb=0)
    L = s.op("ADD", z, bfc)
    M = s.op("MAX", L, a0=1, a1=2)
    E = s.op("EXP", s.op("SUB", L, M))
    P = s.op("DIV", E, s.op("SUM", E, a0=1, a1=2))
    s.output(L, P)
    s.meta["convs"] = net.k
    return s.to_dict()


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}
