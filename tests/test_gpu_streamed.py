"""Streaming a C2 step through the public API in row slices (bench.py's `e2e`).

One graph per row slice, each created on its own caller stream: cg_assign from
pinned host memory, cg_eval and a read-back enqueued on that caller stream must be
ordered by the API's stream joins alone (the graph owns its pool, the
caller owns the stream).  The streamed output must equal the oracle's evaluation
of the whole step, and repeating the step with new inputs must not mix slices or
steps.
"""
import pytest
import torch

from paper_1812_03770_b200 import cg
from tests.gpu_util import normwise, oracle_outputs
from workloads import configs
from workloads.gen import materialise

pytestmark = pytest.mark.gpu


def _data(rows, row0, seed=1812):
    def f(rec):
        if rec["op"] not in ("VAR", "CONST"):
            return None
        shp = rec["shape"]
        off = row0 if (len(shp) == 2 and shp[0] == rows) else 0
        return materialise(rec["data"], shp, seed, row_offset=off)
    return f


def test_c2_streamed_slices_match_oracle():
    rows, cols, nch = 1024, 256, 4
    rc = rows // nch
    full = configs.c2(rows, cols)
    streams = [torch.cuda.Stream() for _ in range(nch)]
    graphs = []
    for i in range(nch):
        g, outs = cg.build_from_spec(configs.c2(rc, cols), device=0, data_fn=_data(rc, i * rc), stream=streams[i].cuda_stream)
        g.optimise(outs)
        g.plan_memory(outs, 0)
        graphs.append((g, outs))
    try:
        hout = torch.empty((rows, cols), dtype=torch.float32).pin_memory()
        for step, seed in enumerate((7, 8)):  # two steps with different inputs
            fdata = _data(rows, 0, seed)
            hx = torch.from_numpy(fdata(full["nodes"][0])).pin_memory()
            hy = torch.from_numpy(fdata(full["nodes"][1])).pin_memory()
            for i, (g, outs) in enumerate(graphs):
                g.assign(0, hx[i * rc:(i + 1) * rc])
                g.assign(1, hy[i * rc:(i + 1) * rc])
                ptr = g.eval(outs)[0]
                with torch.cuda.stream(streams[i]):
                    hout[i * rc:(i + 1) * rc].copy_(g.view(ptr, (rc, cols)), non_blocking=True)
            torch.cuda.synchronize()
            ref, _, _ = oracle_outputs(full, {0: hx.numpy(), 1: hy.numpy()})
            assert normwise(hout.numpy(), ref[full["outputs"][0]]) <= 1e-5, step
    finally:
        for g, _ in graphs:
            g.destroy()
