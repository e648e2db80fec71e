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


C5_CONVS = [  # (N, H, W, Ci, KH, KW, Co, stride, pad) of InceptionV3 at batch 256 (pad 1 = SAME)
    (256, 35, 35, 288, 1, 1, 64, 1, 1), (256, 35, 35, 64, 3, 3, 96, 1, 1), (256, 35, 35, 48, 5, 5, 64, 1, 1),
    (256, 17, 17, 768, 1, 1, 192, 1, 1), (256, 17, 17, 128, 1, 7, 128, 1, 1), (256, 147, 147, 32, 3, 3, 64, 1, 1),
    (256, 149, 149, 32, 3, 3, 32, 1, 0), (256, 299, 299, 3, 3, 3, 32, 2, 0),
    (256, 17, 17, 192, 7, 1, 192, 1, 1), (256, 35, 35, 64, 3, 3, 96, 1, 1),
    (256, 73, 73, 80, 3, 3, 192, 1, 0), (256, 73, 73, 64, 1, 1, 80, 1, 1)]


def conv_main(a):
    sel = [int(i) for i in a.convs.split(",")] if a.convs != "all" else range(len(C5_CONVS))
    for i in sel:
        n, h, w, ci, kh, kw, co, st, pad = C5_CONVS[i]
        g = cg.Graph(0)
        vx, vw = g.var((n, h, w, ci)), g.var((kh, kw, ci, co))
        o = g.add_node("CONV2D", [vx, vw], sh=st, sw=st, pad=pad)
        g.plan_memory([o])
        rng = np.random.default_rng(0)
        g.assign(vx, rng.uniform(-1, 1, (n, h, w, ci)).astype(np.float32))
        g.assign(vw, rng.uniform(-1, 1, (kh, kw, ci, co)).astype(np.float32))
        ms = time_graph(g, [o], a.iters)
        ho = (h - kh) // st + 1 if pad == 0 else (h + st - 1) // st
        wo = (w - kw) // st + 1 if pad == 0 else (w + st - 1) // st
        fl = 2.0 * n * ho * wo * co * kh * kw * ci
        print(json.dumps({"op": "CONV2D", "shape": C5_CONVS[i], "ms": ms, "tflops": fl / ms / 1e9,
                          "gb_s": 4.0 * (n * h * w * ci + n * ho * wo * co) / ms / 1e6}), flush=True)
        g.destroy()


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
    ap.add_argument("--convs", default="", help="C5 conv indices or 'all' (instead of the dots)")
    a = ap.parse_args()
    if a.convs:
        conv_main(a)
        return
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
