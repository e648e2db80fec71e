"""Time single-op graphs through the C ABI (CUDA events on the graph's work stream).

    python tools/bench_ops.py [--iters N]

Prints one JSON line per case: achieved TFLOP/s (dots) next to torch.matmul
(cuBLAS) fp32 and TF32 on the same shapes, for context only.
"""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg  # noqa: E402

C3_DOTS = [  # (M, N, K, ta, tb) of the C3 training step, batch 4096
    (4096, 1024, 784, 0, 0), (4096, 1024, 1024, 0, 0), (784, 1024, 4096, 1, 0),
    (1024, 1024, 4096, 1, 0), (4096, 1024, 1024, 0, 1), (8192, 8192, 8192, 0, 0)]


def time_graph(g, outs, iters):
    ws = torch.cuda.ExternalStream(g.work_stream())
    for _ in range(3):
        g.eval(outs, cg.EVAL_FULL)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(ws)
    for _ in range(iters):
        g.eval(outs, cg.EVAL_FULL)
    e.record(ws)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def time_torch(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--shapes", default="", help="comma-separated indices into C3_DOTS (default: all)")
    ap.add_argument("--no-torch", action="store_true")
    a = ap.parse_args()
    sel = [int(i) for i in a.shapes.split(",")] if a.shapes else range(len(C3_DOTS))
    for (m, n, k, ta, tb) in [C3_DOTS[i] for i in sel]:
        sa = (k, m) if ta else (m, k)
        sb = (n, k) if tb else (k, n)
        g = cg.Graph(0)
        va, vb = g.var(sa), g.var(sb)
        o = g.add_node("DOT", [va, vb], ta=ta, tb=tb)
        g.plan_memory([o])
        rng = np.random.default_rng(0)
        g.assign(va, rng.uniform(-1, 1, sa).astype(np.float32))
        g.assign(vb, rng.uniform(-1, 1, sb).astype(np.float32))
        ms = time_graph(g, [o], a.iters)
        if a.no_torch:
            print(json.dumps({"op": "DOT", "M": m, "N": n, "K": k, "ta": ta, "tb": tb, "ms": ms,
                              "tflops": 2.0 * m * n * k / ms / 1e9}), flush=True)
            g.destroy()
            continue
        A = torch.randn(sa, device="cuda")
        B = torch.randn(sb, device="cuda")
        fa = (lambda: A.T) if ta else (lambda: A)
        fb = (lambda: B.T) if tb else (lambda: B)
        torch.backends.cuda.matmul.allow_tf32 = False
        ms32 = time_torch(lambda: fa() @ fb(), a.iters)
        torch.backends.cuda.matmul.allow_tf32 = True
        mstf = time_torch(lambda: fa() @ fb(), a.iters)
        fl = 2.0 * m * n * k
        print(json.dumps({"op": "DOT", "M": m, "N": n, "K": k, "ta": ta, "tb": tb, "ms": ms,
                          "tflops": fl / ms / 1e9, "cublas_fp32_tflops": fl / ms32 / 1e9,
                          "cublas_tf32_tflops": fl / mstf / 1e9}), flush=True)
        g.destroy()


if __name__ == "__main__":
    main()
