"""Per-node GPU-vs-oracle comparison for one evaluation of a workloads spec.

Every op node is planned as an output (so every value stays readable), the graph
is evaluated once (no update edges) and each node is compared with the oracle's
eager value (normwise error).

    python tools/node_diff.py C3small|C4small|C1|C2small [--top N]
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle.eager import apply_updates, evaluate, leaf_values  # noqa: E402
from oracle.graph import from_spec  # noqa: E402
from paper_1812_03770_b200 import cg  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.gen import materialise, retag  # noqa: E402


def nw(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    m = np.max(np.abs(want))
    return float(np.max(np.abs(got - want)) / m) if m > 0 else float(np.max(np.abs(got)))

SPECS = {
    "C3small": lambda: configs.c3(batch=256, widths=(784, 128, 64, 10)),
    "C4small": lambda: configs.c4(batch=64),
    "C1": lambda: configs.c1(1024),
    "C2small": lambda: configs.c2(rows=64, cols=1024),
    "C5small": lambda: configs.c5(batch=2),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("spec")
    ap.add_argument("--top", type=int, default=15)
    ap.add_argument("--iters", type=int, default=1, help="compare at the last of N training iterations")
    ap.add_argument("--first", type=float, default=0.0, help="also print the first nodes (creation order) above this error")
    a = ap.parse_args()
    spec = SPECS[a.spec]()
    ops = [n["id"] for n in spec["nodes"] if n["op"] not in ("VAR", "CONST")]
    spec = dict(spec, outputs=ops)
    if a.iters <= 1:
        spec["updates"] = []

    def data(rec):
        return materialise(rec["data"], rec["shape"]) if rec["op"] in ("VAR", "CONST") else None

    g, outs = cg.build_from_spec(spec, device=0, data_fn=data)
    g.plan_memory(outs, cg.PLAN_NO_FUSION)
    og, _ = from_spec(spec)
    state = leaf_values(og)
    per = {n["name"]: n["data"] for n in spec["nodes"] if n.get("name") in spec.get("meta", {}).get("per_iteration", [])}
    name_to_id = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    gpu_vars = {}
    for it in range(a.iters):
        for name, d in per.items():
            i = name_to_id[name]
            v = materialise(retag(d, f"{d['tag']}@{it}"), spec["nodes"][i]["shape"])
            state[i] = v
            g.assign(i, v)
        last = it == a.iters - 1
        if last:  # Var values entering the compared iteration
            gpu_vars = {v: g.read(v) for _, v in og.updates}
        g.eval(outs, cg.EVAL_NO_UPDATE if last else 0)
        ref = evaluate(og, state)
        if not last:
            apply_updates(og, ref, state)
    for v, x in gpu_vars.items():
        print(f"var {og.nodes[v].name}: entering err {nw(x, state[v]):.3e}")
    rows = []
    for n in spec["nodes"]:
        if n["op"] in ("VAR", "CONST"):
            continue
        got = g.read(n["id"]).astype(np.float64)
        want = ref[n["id"]].astype(np.float64)
        m = np.max(np.abs(want))
        err = float(np.max(np.abs(got - want)) / m) if m > 0 else float(np.max(np.abs(got)))
        rows.append((err, n["id"], n["op"], n.get("attrs", {}), list(want.shape), n["preds"]))
    for r in sorted(rows, key=lambda t: -t[0])[: a.top]:
        print(f"err {r[0]:.3e}  id {r[1]} {r[2]} {r[3]} shape {r[4]} preds {r[5]}")
    if a.first > 0:
        print("-- first nodes above", a.first)
        for r in [r for r in rows if r[0] > a.first][: a.top]:
            print(f"err {r[0]:.3e}  id {r[1]} {r[2]} {r[3]} shape {r[4]} preds {r[5]}")


if __name__ == "__main__":
    main()
