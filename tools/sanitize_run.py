"""Small end-to-end workload for compute-sanitizer: C1 (incremental), a small C2,
a small C3 training iteration, a tensor-core dot and conv (with a fused epilogue)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.gen import materialise, retag  # noqa: E402


def data(rec):
    return materialise(rec["data"], rec["shape"]) if rec["op"] in ("VAR", "CONST") else None


for spec, flags in ((configs.c1(1024), cg.PLAN_INCREMENTAL), (configs.c2(64, 1024), 0),
                    (configs.c3(batch=256, widths=(784, 128, 64, 10)), 0), (configs.c4(batch=8), 0)):
    g, outs = cg.build_from_spec(spec, device=0, data_fn=data)
    g.optimise(outs)
    g.plan_memory(outs, flags)
    for it in range(2):
        for n in spec["nodes"]:
            if n.get("name") in spec.get("meta", {}).get("per_iteration", []):
                g.assign(n["id"], materialise(retag(n["data"], f"{n['data']['tag']}@{it}"), n["shape"]))
        g.eval(outs)
    g.read(outs[0])
    g.destroy()
rng = np.random.default_rng(0)
g = cg.Graph(0)
x, w, b = g.var([2, 35, 35, 32]), g.var([3, 3, 32, 64]), g.var([64])
y = g.add_node("RELU", [g.add_node("ADD", [g.add_node("CONV2D", [x, w], sh=1, sw=1, pad=1), b])])
a, bb = g.var([300, 200]), g.var([200, 136])
d = g.add_node("DOT", [a, bb], ta=0, tb=0)
info = g.plan_memory([y, d])
for v, s in ((x, [2, 35, 35, 32]), (w, [3, 3, 32, 64]), (b, [64]), (a, [300, 200]), (bb, [200, 136])):
    g.assign(v, rng.standard_normal(s).astype(np.float32))
g.eval([y, d])
g.read(y)
print("sanitize workload ok", info["n_fused"])
