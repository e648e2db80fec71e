python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python - > gpurun_out/sib_bitid.log 2>&1 <<'PY'
import os, sys, numpy as np
sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg
from tests.gpu_util import leaf_data
from workloads import configs
res = []
for env in ({"CG_NO_SIBLING_GEMM": "1"}, {}):
    os.environ.pop("CG_NO_SIBLING_GEMM", None); os.environ.update(env)
    spec = configs.c5(batch=256)
    g, outs = cg.build_from_spec(spec, device=0, data_fn=leaf_data)
    g.optimise(outs); info = g.plan_memory(outs, 0)
    g.eval(outs, cg.EVAL_SYNC)
    res.append([g.read(o) for o in outs])
    print(env, "launches", g.launch_count(), "n_fused", info["n_fused"], flush=True)
    g.destroy()
for a, b in zip(*res):
    d = np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(a)), 1e-30)
    print("bit-identical", np.array_equal(a, b), "normwise", d, flush=True)
PY
