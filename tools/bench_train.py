"""Time training iterations of C3 / C4 (and one C5 inference eval) through the C ABI.

An iteration = cg_assign(X), cg_assign(Y) from pre-staged device buffers (D2D)
+ cg_eval (forward, backward, AllReduce nodes, SGD, update copy), timed with CUDA
events on the graph's work stream.  Prints one JSON line per config.

    python tools/bench_train.py [--configs C3,C4,C5] [--iters N]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.gen import materialise, retag  # noqa: E402


def data(rec):
    return materialise(rec["data"], rec["shape"]) if rec["op"] in ("VAR", "CONST") else None


def run(name, iters):
    spec = {"C3": configs.c3, "C4": configs.c4, "C5": configs.c5}[name]()
    t0 = time.perf_counter()
    g, outs = cg.build_from_spec(spec, device=0, data_fn=data)
    rep = g.optimise(outs)
    info = g.plan_memory(outs, cg.PLAN_FUSED_COLL if os.environ.get("CG_COLL", "fused") == "fused" else 0)
    build_s = time.perf_counter() - t0
    ws = torch.cuda.ExternalStream(g.work_stream())
    per = spec["meta"].get("per_iteration", [])
    name_to_id = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    staged = []
    for it in range(4):
        d = {}
        for nm in per:
            i = name_to_id[nm]
            rec = spec["nodes"][i]
            d[i] = torch.from_numpy(materialise(retag(rec["data"], f"{rec['data']['tag']}@{it}"), rec["shape"])).cuda()
        staged.append(d)

    def step(k):
        for i, t in staged[k % len(staged)].items():
            g.assign(i, t)
        g.eval(outs, cg.EVAL_FULL)

    for k in range(3):
        step(k)
    torch.cuda.synchronize()
    l0 = g.launch_count()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(ws)
    for k in range(iters):
        step(k)
    e.record(ws)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    line = {"config": name, "ms_per_iter": ms, "iters_per_s": 1e3 / ms, "kernels_per_iter": (g.launch_count() - l0) / iters,
            "build_s": build_s, "optimiser": rep,
            "plan": {k: info[k] for k in ("n_groups", "n_blocks", "n_kernels", "pool_bytes", "external_bytes",
                                          "workspace_bytes", "unshared_bytes")}}
    print(json.dumps(line), flush=True)
    g.destroy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C4")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    for c in a.configs.split(","):
        run(c, a.iters)


if __name__ == "__main__":
    main()
