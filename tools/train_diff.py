"""Iteration-by-iteration GPU-vs-oracle comparison of a training spec (loss and
every parameter after each update).

    python tools/train_diff.py C3small|C4small [--iters N] [--flags F]
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle.eager import ancestors, apply_updates, evaluate, leaf_values  # noqa: E402
from oracle.graph import from_spec  # noqa: E402
from paper_1812_03770_b200 import cg  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.gen import materialise, retag  # noqa: E402

SPECS = {
    "C3small": lambda: configs.c3(batch=256, widths=(784, 128, 64, 10)),
    "C3": lambda: configs.c3(),
    "C4small": lambda: configs.c4(batch=64),
}


def nw(got, want):
    got, want = got.astype(np.float64), want.astype(np.float64)
    m = np.max(np.abs(want))
    return float(np.max(np.abs(got - want)) / m) if m > 0 else float(np.max(np.abs(got)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("spec")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--flags", type=int, default=0)
    a = ap.parse_args()
    spec = SPECS[a.spec]()

    def data(rec):
        return materialise(rec["data"], rec["shape"]) if rec["op"] in ("VAR", "CONST") else None

    g, outs = cg.build_from_spec(spec, device=0, data_fn=data)
    g.optimise(outs)
    g.plan_memory(outs, a.flags)
    og, oo = from_spec(spec)
    per = {n["name"]: n["data"] for n in spec["nodes"] if n.get("name") in spec["meta"]["per_iteration"]}
    name_to_id = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    state = leaf_values(og)
    needed = ancestors(og, list(oo) + [u for u, _ in og.updates])
    for it in range(a.iters):
        for name, d in per.items():
            i = name_to_id[name]
            v = materialise(retag(d, f"{d['tag']}@{it}"), spec["nodes"][i]["shape"])
            state[i] = v
            g.assign(i, v)
        g.eval(outs)
        vals = evaluate(og, state, needed)
        apply_updates(og, vals, state)
        msg = [f"it {it} loss {nw(g.read(outs[0]), vals[oo[0]]):.2e} logits {nw(g.read(outs[1]), vals[oo[1]]):.2e}"]
        for u, v in og.updates:
            msg.append(f"{og.nodes[v].name} {nw(g.read(v), state[v]):.2e}")
        print("  ".join(msg), flush=True)


if __name__ == "__main__":
    main()
