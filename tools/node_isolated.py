"""Per-node ISOLATED GPU-vs-oracle error: every op node is an output; each node's
GPU value is compared with the oracle's op applied to the GPU's own input values
(so each kernel's rounding is measured alone, not the errors it inherits).

    python tools/node_isolated.py C4 [batch]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle.graph import from_spec  # noqa: E402
from oracle.eager import leaf_values  # noqa: E402
from oracle.ops import eval_op  # noqa: E402
from tests.gpu_util import gpu_graph  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.gen import materialise, retag  # noqa: E402

name = sys.argv[1]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
spec = configs.c4(batch=batch) if name == "C4" else configs.c3(batch=batch)
spec = dict(spec)
ops = [n["id"] for n in spec["nodes"] if n["op"] not in ("VAR", "CONST")]
spec["outputs"] = ops
spec["updates"] = []
og, _ = from_spec(spec)
leaves = leaf_values(og)
ids = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
g, outs, _, _ = gpu_graph(spec, 0, optimise=False)
for nm in spec["meta"]["per_iteration"]:
    rec = spec["nodes"][ids[nm]]
    leaves[ids[nm]] = materialise(retag(rec["data"], f"{rec['data']['tag']}@0"), rec["shape"])
    g.assign(ids[nm], leaves[ids[nm]])
g.eval(outs)
vals = dict(leaves)
for i in ops:
    vals[i] = g.read(i)
rows = []
for n in og.nodes:
    if n.id not in ops:
        continue
    want = eval_op(n.op, [vals[p] for p in n.preds], n.attrs, n.shape).astype(np.float64)
    got = vals[n.id].astype(np.float64)
    m = np.max(np.abs(want))
    e = float(np.max(np.abs(got - want)) / m) if m > 0 else float(np.max(np.abs(got)))
    rows.append((e, n.id, n.op, tuple(n.shape)))
for e, i, op, shp in sorted(rows, reverse=True):
    print(f"{e:.3e}  node {i:3d} {op:20s} {shp}")
