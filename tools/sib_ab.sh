python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pool_fusion.py -m gpu -q -x -k "c5 or conv or epilogue or concat or zero_copy" > gpurun_out/sib_tests.log 2>&1; echo rc=$? >> gpurun_out/sib_tests.log
timeout 300 python - > gpurun_out/sib_bitid.log 2>&1 <<'PY'
import os, sys, numpy as np
sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg
from tests.gpu_util import leaf_data
from workloads import configs
res = []
for env in ({"CG_NO_SIBLING_GEMM": "1"}, {}):
    os.environ.pop("CG_NO_SIBLING_GEMM", None); os.environ.update(env)
    spec = configs.c5(batch=4)
    g, outs = cg.build_from_spec(spec, device=0, data_fn=leaf_data)
    g.optimise(outs); info = g.plan_memory(outs, 0)
    g.eval(outs, cg.EVAL_SYNC)
    res.append([g.read(o) for o in outs])
    print(env, "launches", g.launch_count(), "n_fused", info["n_fused"])
    g.destroy()
for a, b in zip(*res):
    d = np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(a)), 1e-30)
    print("bit-identical", np.array_equal(a, b), "normwise", d)
PY
for i in 1 2; do
  timeout 300 python tools/bench_train.py --configs C5 --iters 5 | grep ms_per | cut -c1-60
  CG_NO_SIBLING_GEMM=1 timeout 300 python tools/bench_train.py --configs C5 --iters 5 | grep ms_per | cut -c1-60
done > gpurun_out/sib_bench.log 2>&1
