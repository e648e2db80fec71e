import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1812_03770_b200 import cg
n = int(sys.argv[1])
x = np.ones((n, 28, 28, 1), np.float32); dy = np.ones((n, 28, 28, 6), np.float32)
g = cg.Graph(0); vx, vd = g.var(x.shape), g.var(dy.shape)
o = g.add_node("CONV2D_BWD_KERNEL", [vx, vd], sh=1, sw=1, pad=1, kh=5, kw=5)
g.plan_memory([o]); g.assign(vx, x); g.assign(vd, dy); g.eval([o]); print(g.read(o)[:, :, 0, 0])
