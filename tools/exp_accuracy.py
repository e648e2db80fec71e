import os, sys, numpy as np
sys.path.insert(0, '.')
from paper_1812_03770_b200 import cg
x = np.concatenate([np.linspace(-87, 88, 2_000_001, dtype=np.float32), np.random.default_rng(0).standard_normal(1_000_000).astype(np.float32) * 4]).astype(np.float32)
g = cg.Graph(0); v = g.var(x.shape); e = g.add_node("EXP", [v]); g.plan_memory([e]); g.assign(v, x); g.eval([e]); y = g.read(e).astype(np.float64)
ref = np.exp(x.astype(np.float64))
m = (ref > 1.2e-38) & (ref < 3.4e38)
rel = np.abs(y[m] - ref[m]) / ref[m]
ulp = np.abs(y[m] - ref[m]) / np.spacing(ref[m].astype(np.float32)).astype(np.float64)
print(os.environ.get("CG_FAST_EXP", "0"), "max rel", rel.max(), "max ulp", ulp.max(), "mean ulp", ulp.mean())
