"""C5 smoke: build, plan, one evaluation with timings (batch from argv)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg  # noqa: E402
from tests.gpu_util import leaf_data  # noqa: E402
from workloads import configs  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 8
t0 = time.time()
spec = configs.c5(batch=b)
g, outs = cg.build_from_spec(spec, device=0, data_fn=leaf_data)
g.optimise(outs)
print("build", time.time() - t0, flush=True)
info = g.plan_memory(outs, 0)
print("plan", time.time() - t0, info, flush=True)
print("views", g.view_stats(), flush=True)
g.eval(outs, cg.EVAL_SYNC)
print("eval1", time.time() - t0, flush=True)
g.eval(outs, cg.EVAL_SYNC | cg.EVAL_FULL)
print("eval2", time.time() - t0, flush=True)
