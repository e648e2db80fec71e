"""Benchmark of the hot path: evaluate an optimised computation graph on B200.

Default workload (BASELINE.json configs[1], the metric's "fused graph-eval HBM
GB/s"): C2, the 20-op elementwise/broadcast chain on the fixed [2^18, 1024]
fp32 ndarrays, optimised to 17 ops in ONE generated kernel.  A "step" is one
full cg_eval "without reusing pre-computed nodes" (the paper's protocol,
P:385) — CG_EVAL_FULL — with inputs resident in HBM.

Multi-GPU, one process per GPU: C2 is sharded by element range —
rank r owns rows [r*R/P, (r+1)*R/P) of the FIXED global arrays, no collective
("scaling": "strong"); a weak-scaled C2 (every rank its own 2^18 rows) is a
labelled secondary.  C3 / C4 are batch data-parallel (global batch 4096 / 8192
split over the ranks, NCCL AllReduce nodes batched by the executor); C5 is
batch-sharded replicas.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment the script re-launches itself
under torch.distributed.run with N ranks.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
BF16_FALLBACK_TFLOPS = 1650.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d.get("hbm_gbs", HBM_FALLBACK_GBS)),
                "bf16_tflops": float(d.get("bf16_tflops", BF16_FALLBACK_TFLOPS)),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d.get("bf16_tflops", 0.0))),
                "source": "MEASURED_PEAKS.json"}
    return {"hbm_gbs": HBM_FALLBACK_GBS, "bf16_tflops": BF16_FALLBACK_TFLOPS,
            "bf16_tflops_sustained": BF16_FALLBACK_TFLOPS, "source": "B200_PROFILING.md fallback"}


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.p = None
        self.path = os.path.join("/tmp", f"cg_clocks_{os.getpid()}_{device_index}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_distributed(args) -> int:
    """--gpus N without a torchrun environment: run this script under
    torch.distributed.run with N ranks (one per GPU) and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def host_info():
    """Host side of the CPU baseline: core count, BLAS build and thread pools."""
    info = {"os_cpu_count": os.cpu_count(), "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}
    try:
        import numpy as np
        info["numpy"] = np.__version__
        from threadpoolctl import threadpool_info
        info["blas"] = [{"api": p.get("internal_api"), "version": p.get("version"), "threads": p.get("num_threads")}
                        for p in threadpool_info()]
    except Exception as exc:  # noqa: BLE001
        info["blas"] = f"unavailable: {exc}"
    return info


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([p.get("num_threads") or 1 for p in threadpool_info()] or [1])
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------- oracle (CPU) legs
# The oracle is the deliberately plain, slow reference; bench.py
# may execute it only here: the cpu_baseline objects and --impl reference.
def oracle_c2_rate(budget_s=12.0, rows=2048):
    """The oracle as it stands (plain eager f64 interpreter), on a bounded row sample
    of the C2 workload; returns (GB/s algorithmic, sample description, seconds)."""
    from oracle.eager import evaluate, leaf_values
    from oracle.graph import from_spec
    from workloads import configs
    spec = configs.c2(rows=rows)
    og, oo = from_spec(spec)
    vals = leaf_values(og)
    t0 = time.perf_counter()
    n = 0
    while True:
        evaluate(og, vals)
        n += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = (time.perf_counter() - t0) / n
    gbs = configs.c2_algo_bytes(rows) / dt / 1e9
    return gbs, f"C2 chain on a [{rows}, 1024] row sample, {n} eager evals ({dt * 1e3:.1f} ms each)", dt


def oracle_secondary(name):
    """Oracle timing for the training / inference configs on a bounded sample:
    C3 10 full iterations (batch 4096); C4 2 iterations of a 1024-image sub-batch;
    C5 images {0, 255} (inference is independent per image)."""
    from oracle.eager import evaluate, leaf_values, run_iterations
    from oracle.graph import from_spec
    from workloads import configs
    from workloads.gen import materialise
    if name == "C3":
        spec = configs.c3()
        og, oo = from_spec(spec)
        per = {n["name"]: n["data"] for n in spec["nodes"] if n.get("name") in spec["meta"]["per_iteration"]}
        t0 = time.perf_counter()
        run_iterations(og, oo, 10, per)
        dt = (time.perf_counter() - t0) / 10
        return {"value": 1.0 / dt, "unit": "iters/s", "s_per_iter": dt, "sample": "C3 full size, 10 iterations"}
    if name == "C4":
        spec = configs.c4(batch=1024, batch_global=8192)
        og, oo = from_spec(spec)
        per = {n["name"]: n["data"] for n in spec["nodes"] if n.get("name") in spec["meta"]["per_iteration"]}
        t0 = time.perf_counter()
        run_iterations(og, oo, 2, per)
        dt = (time.perf_counter() - t0) / 2 * 8  # 8 sub-batches of 1024 per global-batch iteration
        return {"value": 1.0 / dt, "unit": "iters/s", "s_per_iter": dt,
                "sample": "C4: 2 iterations of a 1024-image sub-batch, scaled x8 to the 8192 batch"}
    spec = configs.c5(batch=2)
    og, oo = from_spec(spec)
    full = configs.c5()
    xs = materialise(full["nodes"][0]["data"], full["nodes"][0]["shape"], rows=[0, 255])
    vals = leaf_values(og, {0: xs})
    t0 = time.perf_counter()
    evaluate(og, vals)
    dt = time.perf_counter() - t0
    return {"value": 2.0 / dt, "unit": "images/s", "s_per_image": dt / 2, "sample": "C5 images {0, 255}"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    per_step = max(1.0, 60.0 / max(1, args.steps + args.warmup))
    gbs, sample, dt = oracle_c2_rate(budget_s=per_step * max(1, args.steps))
    line = {"impl": "reference", "metric": "fused graph-eval HBM GB/s", "value": gbs, "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 compute / fp32 storage",
            "data": "synthetic (seeded splitmix64, SURVEY §8(d))",
            "config": {"workload": "C2 20-op chain (oracle on a row sample)", "rows": 2048, "cols": 1024},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "host": host_info()},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- helpers (CUDA arm)
def plan_traffic_bytes(g) -> int:
    """Algorithmic bytes of one full evaluation of the PLANNED graph: every group
    reads each of its distinct inputs once and writes its materialised values
    once (interior values of fused groups never touch HBM)."""
    plan = json.loads(g.dump_json(1))
    shapes = {}

    def nbytes(v):
        if v not in shapes:
            shapes[v] = 4 * math.prod(g.shape(v))
        return shapes[v]
    return sum(sum(nbytes(p) for p in gr["inputs"]) + sum(nbytes(m) for m in gr["materialised"])
               for gr in plan["groups"])


def graph_flops(g, spec) -> int:
    """Algorithmic FLOPs of the dot / conv nodes: 2*M*N*K per DOT, 2*N*Ho*Wo*Co*KH*KW*Ci
    per convolution (forward, backward-input and backward-kernel alike)."""
    total = 0
    for rec in spec["nodes"]:
        op = rec["op"]
        if op == "DOT":
            m, n = g.shape(rec["id"])
            a = g.shape(rec["preds"][0])
            total += 2 * m * n * (a[0] if rec["attrs"].get("ta") else a[1])
        elif op == "CONV2D":
            kh, kw, ci, co = g.shape(rec["preds"][1])
            nb, ho, wo, _ = g.shape(rec["id"])
            total += 2 * nb * ho * wo * co * kh * kw * ci
        elif op == "CONV2D_BWD_INPUT":
            nb, ho, wo, co = g.shape(rec["preds"][0])
            kh, kw, ci, _ = g.shape(rec["preds"][1])
            total += 2 * nb * ho * wo * co * kh * kw * ci
        elif op == "CONV2D_BWD_KERNEL":
            kh, kw, ci, co = g.shape(rec["id"])
            nb, ho, wo, _ = g.shape(rec["preds"][1])
            total += 2 * nb * ho * wo * co * kh * kw * ci
    return total


def measure_tf32_peak(dev):
    """Dense TF32 tensor throughput (SURVEY §8(d) roofline denominator): torch.matmul
    8192^3 fp32 with TF32 allowed, best of 10 (burst), CUDA events."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        best = float("inf")
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch.matmul(a, b)
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        del a, b
        return 2 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def _all_ok(ok, world):
    """MIN over ranks of a per-rank success flag: a failure on one rank skips the
    rest of the secondary configs on EVERY rank (no rank left waiting in a collective)."""
    if world == 1:
        return ok
    import torch
    import torch.distributed as dist
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t[0])


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _launches_of(g, fn):
    """Kernel launches of ONE step (counted by the engine around a single extra call,
    so warm-up and load-phase steps do not enter the figure)."""
    l0 = g.launch_count()
    fn(0)
    return g.launch_count() - l0


def _timed(ws, fn, iters, world, local, min_s=0.6):
    """Warm-up, a load phase of >= 0.3 s (so the sampled clocks are this kernel
    mix's clocks), then `iters` steps (raised to fill >= min_s) timed with CUDA
    events on the graph's work stream between barriers + synchronize; returns
    (ms per step over ranks' max, clocks, iters)."""
    import torch
    for k in range(3):
        fn(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn(0)
    torch.cuda.synchronize()
    est = max(time.perf_counter() - t0, 1e-5)
    iters = max(iters, int(min_s / est))
    iters = int(_max_over_ranks(iters, world))
    clk = Clocks(local).start()
    t_end = time.perf_counter() + 0.3
    k = 0
    while time.perf_counter() < t_end:
        fn(k)
        k += 1
        if k % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(ws)
    for k in range(iters):
        fn(k)
    e.record(ws)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    clocks = clk.stop()
    _barrier(world)
    return _max_over_ranks(ms, world), clocks, iters


# ---------------------------------------------------------------------------- CUDA arm: C2 (primary)
E2E_CHUNKS = int(os.environ.get("CG_E2E_CHUNKS", "8"))  # row slices of the streamed end-to-end step


def build_c2(rows_local, row0, local, stream=None):
    from paper_1812_03770_b200 import cg
    from workloads import configs
    from workloads.gen import materialise
    cols = configs.C2_COLS
    spec = configs.c2(rows_local, cols)

    def data(rec):
        if rec["op"] not in ("VAR", "CONST"):
            return None
        shp = rec["shape"]
        off = row0 if (len(shp) == 2 and shp[0] == rows_local) else 0
        return materialise(rec["data"], shp, row_offset=off)
    t0 = time.perf_counter()
    g, outs = cg.build_from_spec(spec, device=local, data_fn=data, stream=stream)
    t_gen = time.perf_counter()
    rep = g.optimise(outs)
    info = g.plan_memory(outs, 0)
    build_s = time.perf_counter() - t_gen
    return g, outs, spec, data, rep, info, build_s, t_gen - t0


def run_c2(args):
    import torch
    import torch.distributed as dist

    from paper_1812_03770_b200 import build as _build
    _build.build()
    from paper_1812_03770_b200 import cg
    from paper_1812_03770_b200.dist import shard_range
    from workloads import configs

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        # a bounded timeout: a rank that fails outside a collective must not leave the
        # others blocked forever (the per-config MIN flag covers the common case)
        import datetime
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(seconds=300))
    rows_g, cols = configs.C2_ROWS, configs.C2_COLS
    row0, rows = shard_range(rows_g, rank, world)  # strong scaling: a slice of the FIXED global arrays
    g, outs, spec, data, rep, info, build_s, gen_s = build_c2(rows, row0, local)
    ws = torch.cuda.ExternalStream(g.work_stream(), device=torch.device("cuda", local))
    algo_local = configs.c2_algo_bytes(rows, cols)
    algo_total = sum(configs.c2_algo_bytes(shard_range(rows_g, r, world)[1], cols) for r in range(world))
    torch.cuda.synchronize()
    for _ in range(max(3, args.warmup)):
        g.eval(outs, cg.EVAL_FULL)
    torch.cuda.synchronize()
    _barrier(world)
    clocks = Clocks(local).start()
    # keep the GPU under this same load for ~0.5 s before the timed region so the
    # sampled clocks are the clocks of the measured kernel (nvidia-smi samples every 100 ms)
    t_end = time.perf_counter() + 0.5
    while time.perf_counter() < t_end:
        for _ in range(20):
            g.eval(outs, cg.EVAL_FULL)
        torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    l0 = g.launch_count()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k_s, k_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_ev.record()
    k_s.record(ws)
    for _ in range(args.steps):
        g.eval(outs, cg.EVAL_FULL)
    k_e.record(ws)
    e_ev.record()
    torch.cuda.synchronize()
    launches = g.launch_count() - l0
    ms = s_ev.elapsed_time(e_ev) / args.steps
    kernel_ms = k_s.elapsed_time(k_e) / args.steps
    clk = clocks.stop()
    _barrier(world)
    ms_max = _max_over_ranks(ms, world)
    kernel_ms_max = _max_over_ranks(kernel_ms, world)
    value = algo_total / (ms_max * 1e-3) / 1e9

    # e2e: through the public API with HOST buffers (pinned), copies inside the timed region
    e2e_steps = max(1, min(args.steps, 3))
    hx = torch.from_numpy(data(spec["nodes"][0])).pin_memory()
    hy = torch.from_numpy(data(spec["nodes"][1])).pin_memory()
    hout = torch.empty((rows, cols), dtype=torch.float32).pin_memory()
    _barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        g.assign(0, hx)
        g.assign(1, hy)
        g.eval(outs)
        g.read_into(outs[0], hout)
    torch.cuda.synchronize()
    e2e_serial_ms = _max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps, world)
    serial_out = hout.clone()
    g.destroy()
    # The same step streamed: the rows in E2E_CHUNKS slices, one graph per slice (its
    # own stream and per-row constants), each slice assign(x, y) -> eval -> D2H of
    # its output on the graph's stream, so slice i's read-back overlaps slice i+1's
    # upload (PCIe is full duplex).  Same public calls, same bytes, same arithmetic.
    nch = E2E_CHUNKS if rows % E2E_CHUNKS == 0 else 1
    rc = rows // nch
    # each slice graph's caller stream is its own torch stream: cg_assign / cg_eval
    # join it both ways, so the read-back enqueued there follows the eval and the next
    # step's upload follows the read-back, with no ordering between slices
    sstreams = [torch.cuda.Stream(device=torch.device("cuda", local)) for _ in range(nch)]
    chunks = [build_c2(rc, row0 + i * rc, local, stream=sstreams[i].cuda_stream)[:2] for i in range(nch)]

    def streamed_step():
        for i, (cg_, couts) in enumerate(chunks):
            cg_.assign(0, hx[i * rc:(i + 1) * rc])
            cg_.assign(1, hy[i * rc:(i + 1) * rc])
            ptr = cg_.eval(couts)[0]
            with torch.cuda.stream(sstreams[i]):
                hout[i * rc:(i + 1) * rc].copy_(cg_.view(ptr, (rc, cols)), non_blocking=True)

    streamed_step()  # (first use of each slice graph outside the timed region)
    torch.cuda.synchronize()
    hout.zero_()
    _barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        streamed_step()
    torch.cuda.synchronize()
    e2e_ms = _max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps, world)
    e2e_val = algo_total / (e2e_ms * 1e-3) / 1e9
    assert torch.equal(hout, serial_out), "streamed e2e output differs from the one-graph step"
    for cg_, _ in chunks:
        cg_.destroy()
    del hx, hy, hout, serial_out

    secondary = None
    if not args.no_secondary:
        try:  # (the C2 line above is printed whatever happens to the secondary configs)
            secondary = run_secondary(rank, world, local, max(5, args.steps), args)
        except Exception as exc:  # noqa: BLE001
            import traceback
            traceback.print_exc(file=sys.stderr)
            secondary = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if rank == 0:
        pk = peaks()
        achieved = algo_local / (kernel_ms * 1e-3) / 1e9  # rank 0's kernel: its own bytes / its own time
        traffic = None
        tp = os.path.join(ROOT, "profiles", "c2_traffic.json")
        if os.path.exists(tp):
            tj = json.load(open(tp))
            # ncu captures the single-GPU kernel (2^28 elements); scale to this rank's shard
            traffic = tj.get("dram_bytes_per_launch") * rows / rows_g if tj.get("dram_bytes_per_launch") else None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            gbs, sample, _ = oracle_c2_rate(budget_s=args.cpu_budget)
            cpu = {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                   "host": host_info()}
        line = {
            "metric": "fused graph-eval HBM GB/s", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded splitmix64)",
            "config": {"workload": "C2: 20-op elementwise/broadcast chain (CSE+CF -> 17 ops, 1 fused kernel)",
                       "global_rows": rows_g, "cols": cols, "elements": rows_g * cols, "rows_per_gpu": rows,
                       "algorithmic_bytes_per_step": algo_total, "parallelism": f"element-range x{world} (no collective)",
                       "l2": "3 GiB moved per step >> 126 MB L2: no flush needed",
                       "eval": "CG_EVAL_FULL (no reuse of pre-computed nodes, P:385)",
                       "build_s": build_s, "optimiser": rep,
                       "plan": {k: info[k] for k in ("n_groups", "n_blocks", "pool_bytes", "unshared_bytes")}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "peak_source": pk["source"],
                         "kernel_ms": kernel_ms, "kernel_ms_max_over_ranks": kernel_ms_max},
            "clocks": clk,
            "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": 2 * rows * cols * 4 * world,
                    "d2h_bytes_per_step": rows * cols * 4 * world, "ms_per_step": e2e_ms,
                    "pipeline": f"{nch} row slices, one graph (and caller stream) each: uploads, evals and read-backs of different slices overlap",
                    "serial": {"value": algo_total / (e2e_serial_ms * 1e-3) / 1e9, "ms_per_step": e2e_serial_ms,
                               "note": "one graph: assign x, assign y, eval, read, back to back"}},
            "gpu_launches": launches,
            "cpu_baseline": cpu,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- secondary workloads
def run_secondary(rank, world, local, iters, args):
    """BASELINE.json's other metrics: C1 full / incremental eval latency; C3 / C4
    data-parallel training iterations/s (global batch fixed: strong; at N > 1 also
    per-GPU batch fixed: weak); C5 images/s with plan peak bytes vs unshared; at
    N > 1 a weak-scaled C2.  Each carries its own clocks and, where it applies, a
    roofline over the whole step and an oracle timing (rank 0, N = 1)."""
    out = {}
    pk = peaks()
    import torch
    tf32 = None
    try:
        tf32 = measure_tf32_peak(torch.device("cuda", local))
    except Exception as exc:  # noqa: BLE001
        out["tf32_peak_error"] = str(exc)[:200]
    out["peaks"] = {"tf32_tflops_measured": tf32, "hbm_gbs": pk["hbm_gbs"], "source": pk["source"],
                    "tf32_how": "torch.matmul 8192^3 fp32, allow_tf32, best of 10"}
    jobs = [("C1", _sec_c1), ("C3", lambda: _sec_train("C3", 4096, False)),
            ("C4", lambda: _sec_train("C4", 8192, False)), ("C5", _sec_c5)]
    if world > 1:
        jobs += [("C2_weak", _sec_c2_weak), ("C3_weak", lambda: _sec_train("C3", 4096, True)),
                 ("C4_weak", lambda: _sec_train("C4", 8192, True))]
    ctx = {"rank": rank, "world": world, "local": local, "iters": iters, "tf32": tf32, "pk": pk,
           "coll": getattr(args, "coll", "fused")}
    for name, fn in jobs:
        ok = True
        try:
            _CTX.update(ctx)
            out[name] = fn()
        except Exception as exc:  # noqa: BLE001
            import traceback
            traceback.print_exc(file=sys.stderr)
            out[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            ok = False
        try:
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001  (a sticky device error: no further device work here)
            out[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            out["skipped_after"] = name
            break
        if not _all_ok(ok, world):
            out["skipped_after"] = name
            break
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        for name in ("C3", "C4", "C5"):
            if isinstance(out.get(name), dict) and "error" not in out[name]:
                try:
                    cb = oracle_secondary(name)
                    cb.update({"kind": "oracle", "cores": blas_threads(),
                               "cores_note": "numpy f64; DOT/CONV through the BLAS thread pool, elementwise 1 core"})
                    out[name]["cpu_baseline"] = cb
                except Exception as exc:  # noqa: BLE001
                    out[name]["cpu_baseline"] = {"error": str(exc)[:200]}
    return out


_CTX: dict = {}


def _leaf(rec, off=0):
    from workloads.gen import materialise
    if rec["op"] not in ("VAR", "CONST"):
        return None
    return materialise(rec["data"], rec["shape"], row_offset=off)


def _sec_c1():
    import torch

    from paper_1812_03770_b200 import cg
    from workloads import configs
    from workloads.gen import materialise, retag
    local, world = _CTX["local"], _CTX["world"]
    dev = torch.device("cuda", local)
    spec = configs.c1(1024)
    t0 = time.perf_counter()
    g, outs = cg.build_from_spec(spec, device=local, data_fn=_leaf)
    g.plan_memory(outs, cg.PLAN_INCREMENTAL)
    build_s = time.perf_counter() - t0
    ws = torch.cuda.ExternalStream(g.work_stream(), device=dev)
    x3 = [torch.from_numpy(materialise(retag(spec["nodes"][3]["data"], f"x3#{k}"), [1024])).to(dev) for k in range(2)]
    full_ms, clk, _ = _timed(ws, lambda k: g.eval(outs, cg.EVAL_FULL), 200, world, local, min_s=0.3)

    def inc(k):
        g.assign(3, x3[k % 2])
        g.eval(outs)
    inc_ms, _, _ = _timed(ws, inc, 200, world, local, min_s=0.3)
    r = {"metric": "eval latency", "unit": "us", "full_eval_us": full_ms * 1e3,
         "incremental_eval_us (assign x3 + eval)": inc_ms * 1e3, "x2_evaluations": g.eval_count(2),
         "x5_evaluations": g.eval_count(5), "build_s": build_s, "clocks": clk,
         "roofline": {"bound": "launch latency", "note": "12 KiB per eval: HBM time ~2 ns (SURVEY §8(d))"}}
    g.destroy()
    return r


def _sec_train(name, gb, weak):
    import torch

    from paper_1812_03770_b200 import cg
    from paper_1812_03770_b200.dist import dp_spec, make_graph, shard_range
    from workloads import configs
    from workloads.gen import materialise, retag
    rank, world, local = _CTX["rank"], _CTX["world"], _CTX["local"]
    dev = torch.device("cuda", local)
    fn = configs.c3 if name == "C3" else configs.c4
    if weak:  # per-GPU batch fixed at gb, global batch gb * world
        spec = fn(batch=gb, batch_global=gb * world)
        start = rank * gb
        count = gb
    else:
        spec = dp_spec(fn, gb, rank, world)
        start, count = shard_range(gb, rank, world)
    t0 = time.perf_counter()
    fused = _CTX.get("coll", "fused") == "fused"
    g = make_graph(local, world, rank, fused=fused)
    for rec in spec["nodes"]:
        data = _leaf(rec)
        if rec["op"] in ("VAR", "CONST"):
            g.add_node(rec["op"], (), dims=rec["shape"], **({"data": data} if data is not None else {}))
        else:
            g.add_node(rec["op"], rec["preds"], **rec.get("attrs", {}))
    for u, v in spec["updates"]:
        g.add_update(u, v)
    outs = spec["outputs"]
    g.optimise(outs)
    info = g.plan_memory(outs, cg.PLAN_FUSED_COLL if fused else 0)
    if fused and world > 1:
        from paper_1812_03770_b200.dist import connect_fused
        connect_fused(g)
    build_s = time.perf_counter() - t0
    ws = torch.cuda.ExternalStream(g.work_stream(), device=dev)
    ids = {n["name"]: n["id"] for n in spec["nodes"] if n["op"] == "VAR"}
    staged = []
    for it in range(4):
        d = {}
        for nm in spec["meta"]["per_iteration"]:
            rec = spec["nodes"][ids[nm]]
            d[ids[nm]] = torch.from_numpy(materialise(retag(rec["data"], f"{rec['data']['tag']}@{it}"),
                                                      rec["shape"], row_offset=start)).to(dev)
        staged.append(d)

    def step(k):
        for i, t in staged[k % 4].items():
            g.assign(i, t)
        g.eval(outs, cg.EVAL_FULL)
    ms, clk, n = _timed(ws, step, _CTX["iters"], world, local)
    launches_per_iter = _launches_of(g, step)
    flops = graph_flops(g, spec)
    traffic = plan_traffic_bytes(g)
    ms_s = ms * 1e-3
    r = {"metric": "train iters/s", "value": 1e3 / ms, "unit": "iters/s", "ms_per_iter": ms,
         "global_batch": gb * world if weak else gb, "local_batch": count, "scaling": "weak" if weak else "strong",
         "parallelism": f"dp{world}" + ((" (fused peer-memory AllReduce + SGD, one launch per step)" if fused else
                                          " (NCCL AllReduce nodes, batched per step)") if world > 1 else ""),
         "collectives": "fused (AllReduce + SGD update in one kernel, CG_PLAN_FUSED_COLL)" if fused else "nccl",
         "n_fused": info["n_fused"],
         "build_s": build_s, "clocks": clk, "launches_per_iter": launches_per_iter,
         "plan_peak_bytes": info["pool_bytes"] + info["external_bytes"] + info["workspace_bytes"],
         "unshared_bytes": info["unshared_bytes"] + info["external_bytes"],
         "algorithmic_flops_per_iter": flops, "plan_traffic_bytes_per_iter": traffic,
         "collective_batches": g.coll_batches() if world > 1 else 0}
    pk, tf32 = _CTX["pk"], _CTX["tf32"]
    hbm_frac = traffic / ms_s / 1e9 / pk["hbm_gbs"]
    if name == "C3" and tf32:
        ach = 3 * flops / ms_s / 1e12
        r["roofline"] = {"bound": "tensor", "scope": "whole iteration (dots dominate)", "achieved": ach,
                         "peak": tf32, "unit": "TFLOP/s", "frac": ach / tf32,
                         "note": "3xTF32: 3 tensor-core passes per algorithmic FLOP; peak = measured TF32",
                         "hbm_frac_of_plan_traffic": hbm_frac}
    else:
        r["roofline"] = {"bound": "hbm", "scope": "whole iteration", "achieved": traffic / ms_s / 1e9,
                         "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": hbm_frac,
                         "note": "plan traffic = each group reads its inputs and writes its materialised values once"}
    g.destroy()
    return r


def _sec_c5():
    import torch

    from paper_1812_03770_b200 import cg
    from workloads import configs
    world, local = _CTX["world"], _CTX["local"]
    dev = torch.device("cuda", local)
    spec = configs.c5()
    t0 = time.perf_counter()
    g, outs = cg.build_from_spec(spec, device=local, data_fn=_leaf)
    g.optimise(outs)
    info = g.plan_memory(outs, 0)
    build_s = time.perf_counter() - t0
    ws = torch.cuda.ExternalStream(g.work_stream(), device=dev)
    ms, clk, n = _timed(ws, lambda k: g.eval(outs, cg.EVAL_FULL), max(2, _CTX["iters"] // 4), world, local)
    launches = _launches_of(g, lambda k: g.eval(outs, cg.EVAL_FULL))
    peak = info["pool_bytes"] + info["external_bytes"] + info["workspace_bytes"]
    unshared = info["unshared_bytes"] + info["external_bytes"]
    flops = graph_flops(g, spec)
    tf32 = _CTX["tf32"]
    r = {"metric": "images/s", "value": world * 256 / (ms * 1e-3), "unit": "images/s", "ms_per_eval": ms,
         "batch_per_gpu": 256, "scaling": "weak", "plan_peak_bytes": peak, "unshared_bytes": unshared,
         "peak_vs_unshared": peak / unshared, "n_groups": info["n_groups"], "n_blocks": info["n_blocks"],
         "build_s": build_s, "clocks": clk, "launches_per_eval": launches, "algorithmic_flops_per_eval": flops,
         "n_fused_epilogues": info["n_fused"],
         "zero_copy_concat_slices": g.view_stats()}  # R14: direct = stored by the conv epilogue
    if tf32:
        ach = 3 * flops / (ms * 1e-3) / 1e12
        r["roofline"] = {"bound": "tensor", "scope": "whole evaluation (convs dominate)", "achieved": ach,
                         "peak": tf32, "unit": "TFLOP/s", "frac": ach / tf32,
                         "note": "3xTF32: 3 tensor-core passes per algorithmic FLOP; peak = measured TF32"}
    g.destroy()
    return r


def _sec_c2_weak():
    import torch

    from paper_1812_03770_b200 import cg
    from workloads import configs
    rank, world, local = _CTX["rank"], _CTX["world"], _CTX["local"]
    rows = configs.C2_ROWS
    g, outs, _, _, _, _, build_s, _ = build_c2(rows, rank * rows, local)
    ws = torch.cuda.ExternalStream(g.work_stream(), device=torch.device("cuda", local))
    ms, clk, _ = _timed(ws, lambda k: g.eval(outs, cg.EVAL_FULL), 20, world, local)
    algo = configs.c2_algo_bytes(rows)
    g.destroy()
    return {"metric": "fused graph-eval HBM GB/s", "value": world * algo / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "ms_per_step": ms, "scaling": "weak", "rows_per_gpu": rows, "clocks": clk, "build_s": build_s}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--coll", default="fused", choices=["fused", "nccl"],
                    help="C3/C4 gradient AllReduce: fused peer-memory kernel with the SGD update (default) or NCCL")
    ap.add_argument("--no-secondary", action="store_true", help="C2 only (skip the C1/C3/C4/C5 lines)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(relaunch_distributed(args))
    run_c2(args)


if __name__ == "__main__":
    main()
