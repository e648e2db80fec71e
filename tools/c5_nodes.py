"""Per-node check of the full-size C5 graph (batch 256) on images {0, 255}:
every op node is an output, rows 0 and 255 of each value are sliced on the
device and compared with the oracle evaluated on those two images.

    python tools/c5_nodes.py [--flags F] [--no-optimise] [--first 1e-4] [--repeat]
"""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.eager import evaluate, leaf_values  # noqa: E402
from oracle.graph import from_spec  # noqa: E402
from paper_1812_03770_b200 import cg  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.gen import materialise  # noqa: E402


def nw(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    m = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / m) if m > 0 else float(np.max(np.abs(a)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--no-optimise", action="store_true")
    ap.add_argument("--first", type=float, default=1e-4)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--repeat", action="store_true", help="evaluate twice and report non-deterministic nodes")
    ap.add_argument("--probe", default="", help="comma list of op names whose nodes become extra outputs "
                    "(the rest keep the shared-block plan); default: every op node is an output")
    ap.add_argument("--ids", default="", help="comma list of node ids to make extra outputs")
    a = ap.parse_args()
    B = a.batch
    spec = configs.c5(batch=B)
    if a.ids:
        ops = list(spec["outputs"]) + [int(x) for x in a.ids.split(",")]
    elif a.probe:
        kinds = set(a.probe.split(","))
        ops = list(spec["outputs"]) + [n["id"] for n in spec["nodes"] if n["op"] in kinds]
    else:
        ops = [n["id"] for n in spec["nodes"] if n["op"] not in ("VAR", "CONST")]
    spec = dict(spec, outputs=ops)
    rows = [0, B - 1]

    def data(rec):
        return materialise(rec["data"], rec["shape"]) if rec["op"] in ("VAR", "CONST") else None

    g, outs = cg.build_from_spec(spec, device=0, data_fn=data)
    if not a.no_optimise:
        g.optimise(outs)
    g.plan_memory(outs, a.flags)

    def snap():
        ptrs = g.eval(outs, cg.EVAL_FULL)
        torch.cuda.synchronize()
        got = {}
        for i, p in zip(outs, ptrs):
            shp = g.shape(i)
            t = g.view(p, shp)
            got[i] = t[rows].cpu().numpy() if shp[0] == B else t.cpu().numpy()
        return got

    got = snap()
    if a.repeat:
        again = snap()
        bad = [i for i in outs if not np.array_equal(got[i], again[i])]
        print("non-deterministic nodes:", len(bad), bad[:20])
    small = configs.c5(batch=2)
    og, _ = from_spec(small)
    xs = materialise(spec["nodes"][0]["data"], spec["nodes"][0]["shape"], rows=rows)
    ref = evaluate(og, leaf_values(og, {0: xs}))
    shown = 0
    for n in spec["nodes"]:
        i = n["id"]
        if n["op"] in ("VAR", "CONST") or i not in got:
            continue
        want = ref[i]
        have = got[i] if got[i].shape == want.shape else None
        if have is None:
            continue
        e = nw(have, want)
        if n["op"] == "CONCAT" and e > a.first:
            off = 0
            for pidx in n["preds"]:
                c = ref[pidx].shape[-1]
                print(f"    segment pred {pidx} channels [{off},{off + c}): err {nw(have[..., off:off + c], want[..., off:off + c]):.3e}"
                      f"  rows: " + " ".join(f"{nw(have[r, ..., off:off + c], want[r, ..., off:off + c]):.1e}" for r in range(2)))
                off += c
        if e > a.first or (a.ids and str(i) in a.ids.split(",")):
            print(f"err {e:.3e} id {i} {n['op']} {n.get('attrs', {})} shape {g.shape(i)} preds {n['preds']}")
            shown += 1
            if shown >= 15:
                break


if __name__ == "__main__":
    main()
