"""C4 at batch 8192: per-iteration GPU-vs-oracle errors, free-running and
teacher-forced (each iteration from the oracle's parameter state).  Diagnostic."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.eager import ancestors, apply_updates, evaluate, leaf_values  # noqa: E402
from oracle.graph import from_spec  # noqa: E402
from tests.gpu_util import gpu_graph, normwise  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.gen import materialise, retag  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
spec = configs.c4(batch=batch)
og, oo = from_spec(spec)
per = {n["name"]: n["data"] for n in spec["nodes"] if n.get("name") in spec["meta"]["per_iteration"]}
ids = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
state = leaf_values(og)
needed = ancestors(og, list(oo) + [u for u, _ in og.updates])
snaps, hist, inputs = [], [], []
for it in range(iters):
    d = {}
    for name, sp in per.items():
        i = ids[name]
        state[i] = materialise(retag(sp, f"{sp['tag']}@{it}"), og.nodes[i].shape)
        d[i] = state[i]
    inputs.append(d)
    snaps.append({v: state[v].copy() for _, v in og.updates})
    vals = evaluate(og, state, needed)
    hist.append({o: vals[o] for o in oo})
    apply_updates(og, vals, state)
    print("oracle it", it, flush=True)
g, outs, _, _ = gpu_graph(spec, 0)
names = {v: og.nodes[v].name for _, v in og.updates}
for it in range(iters):
    for i, x in inputs[it].items():
        g.assign(i, x)
    g.eval(outs)
    print(f"free it {it}: loss rel {abs(float(g.read(outs[0]).ravel()[0]) / float(hist[it][oo[0]].ravel()[0]) - 1):.2e}"
          f" logits {normwise(g.read(outs[1]), hist[it][oo[1]]):.2e}", flush=True)
print("free final:", {names[v]: f"{normwise(g.read(v), state[v]):.2e}" for _, v in og.updates})
g2, outs2, _, _ = gpu_graph(spec, 0)
for it in range(iters):
    for i, x in inputs[it].items():
        g2.assign(i, x)
    for v, x in snaps[it].items():
        g2.assign(v, x)
    g2.eval(outs2)
    nxt = snaps[it + 1] if it + 1 < iters else {v: state[v] for _, v in og.updates}
    print(f"teacher it {it}: logits {normwise(g2.read(outs2[1]), hist[it][oo[1]]):.2e} ",
          {names[v]: f"{normwise(g2.read(v), nxt[v]):.1e}" for _, v in og.updates}, flush=True)
