"""C5 (batch 256) logits of images {0, 255} vs the oracle under plan variants.

    python tools/c5_check.py [--batch B]
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


def nw(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    a = ap.parse_args()
    B = a.batch
    spec = configs.c5(batch=B)
    rows = [0, B - 1]
    og, oo = from_spec(configs.c5(batch=2))
    xs = materialise(spec["nodes"][0]["data"], spec["nodes"][0]["shape"], rows=rows)
    ref = evaluate(og, leaf_values(og, {0: xs}))

    def data(rec):
        return materialise(rec["data"], rec["shape"]) if rec["op"] in ("VAR", "CONST") else None

    for opt in (True, False):
        for flags in (0, cg.PLAN_NO_FUSION):
            g, outs = cg.build_from_spec(spec, device=0, data_fn=data)
            if opt:
                g.optimise(outs)
            g.plan_memory(outs, flags)
            g.eval(outs)
            L = g.read(outs[0])
            print(f"optimise={opt} flags={flags}: " + "  ".join(
                f"img{r} logits {nw(L[r], ref[oo[0]][i]):.2e}" for i, r in enumerate(rows)), flush=True)
            g.destroy()


if __name__ == "__main__":
    main()
