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
from oracle.eager import evaluate, leaf_values  # noqa: E402
from oracle.graph import from_spec  # noqa: E402
from paper_1812_03770_b200 import cg  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.gen import materialise  # noqa: E402

SPECS = {
    "C3small": lambda: configs.c3(batch=256, widths=(784, 128, 64, 10)),
    "C4small": lambda: configs.c4(batch=64),
    "C1": lambda: configs.c1(1024),
    "C2small": lambda: configs.c2(rows=64, cols=1024),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("spec")
    ap.add_argument("--top", type=int, default=15)
    a = ap.parse_args()
    spec = SPECS[a.spec]()
    ops = [n["id"] for n in spec["nodes"] if n["op"] not in ("VAR", "CONST")]
    spec = dict(spec, outputs=ops, updates=[])

    def data(rec):
        return materialise(rec["data"], rec["shape"]) if rec["op"] in ("VAR", "CONST") else None

    g, outs = cg.build_from_spec(spec, device=0, data_fn=data)
    g.plan_memory(outs, cg.PLAN_NO_FUSION)
    g.eval(outs)
    og, _ = from_spec(spec)
    ref = evaluate(og, leaf_values(og))
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


if __name__ == "__main__":
    main()
