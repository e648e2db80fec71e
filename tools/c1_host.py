import sys, time
sys.path.insert(0, ".")
import torch
from paper_1812_03770_b200 import cg
from workloads import configs
from workloads.gen import materialise, retag
spec = configs.c1(1024)
def leaf(rec, off=0):
    return materialise(rec["data"], rec["shape"]) if rec["op"] in ("VAR", "CONST") else None
g, outs = cg.build_from_spec(spec, device=0, data_fn=leaf)
g.plan_memory(outs, cg.PLAN_INCREMENTAL)
x3 = [torch.from_numpy(materialise(retag(spec["nodes"][3]["data"], f"x3#{k}"), [1024])).cuda() for k in range(2)]
for _ in range(10):
    g.eval(outs, cg.EVAL_FULL)
torch.cuda.synchronize()
for name, fn in [("assign", lambda k: g.assign(3, x3[k % 2])), ("eval_inc", lambda k: g.eval(outs)),
                 ("assign+eval", lambda k: (g.assign(3, x3[k % 2]), g.eval(outs))), ("eval_full", lambda k: g.eval(outs, cg.EVAL_FULL))]:
    for k in range(50): fn(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(2000): fn(k)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(name, (t1 - t0) / 2000 * 1e6, "us host per call")
