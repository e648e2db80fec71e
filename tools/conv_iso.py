"""Time one C4 conv (+ bias epilogue) in isolation: python tools/conv_iso.py [conv1|conv2] [iters]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "conv1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
n = 8192
xs, ws, pad = ((n, 28, 28, 1), (5, 5, 1, 6), 1) if which == "conv1" else ((n, 14, 14, 6), (5, 5, 6, 16), 0)
rng = np.random.default_rng(0)
g = cg.Graph(0)
vx, vw, vb = g.var(xs), g.var(ws), g.var((1, 1, 1, ws[3]))
y = g.add_node("CONV2D", [vx, vw], sh=1, sw=1, pad=pad)
out = g.add_node("ADD", [y, vb])
info = g.plan_memory([out])
g.assign(vx, rng.uniform(-1, 1, xs).astype(np.float32))
g.assign(vw, rng.uniform(-1, 1, ws).astype(np.float32))
g.assign(vb, rng.uniform(-1, 1, (1, 1, 1, ws[3])).astype(np.float32))
for _ in range(3):
    g.eval([out], cg.EVAL_FULL)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    g.eval([out], cg.EVAL_FULL)
e1.record()
torch.cuda.synchronize()
print(f"{which} n_fused={info['n_fused']} us_per_eval={e0.elapsed_time(e1) * 1000 / iters:.1f}")
