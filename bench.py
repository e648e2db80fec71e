"""Benchmark of the hot path: evaluate an optimised computation graph on B200.

Default workload (BASELINE.json configs[1], the metric's "fused graph-eval HBM
GB/s"): C2, the 20-op elementwise/broadcast chain on a [2^18, 1024] fp32
ndarray per GPU, optimised to 17 ops in ONE generated kernel.  A "step" is
one full cg_eval "without reusing pre-computed nodes" (the paper's protocol,
P:385) — CG_EVAL_FULL — with inputs resident in HBM.  Multi-GPU: element-range
sharding (each rank owns its own [2^18, 1024] row range of an N x larger
global array; no collective on the data path) => "scaling": "weak".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2|C1|C3|C4]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", HBM_FALLBACK_GBS)), "measured"
    return HBM_FALLBACK_GBS, "fallback"


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.p = None
        self.path = os.path.join("/tmp", f"cg_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

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
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------- oracle (CPU) arm
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


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    per_step = max(1.0, 60.0 / max(1, args.steps + args.warmup))
    gbs, sample, dt = oracle_c2_rate(budget_s=per_step * max(1, args.steps))
    line = {"impl": "reference", "metric": "fused graph-eval HBM GB/s", "value": gbs, "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 compute / fp32 storage",
            "data": "synthetic (seeded splitmix64, SURVEY §8(d))",
            "config": {"workload": "C2 20-op chain (oracle on a row sample)", "rows": 2048, "cols": 1024},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- CUDA arm: C2
def run_c2(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1812_03770_b200 import build as _build
    _build.build()
    from paper_1812_03770_b200 import cg
    from workloads import configs
    from workloads.gen import materialise

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rows, cols = configs.C2_ROWS, configs.C2_COLS
    spec = configs.c2(rows, cols)
    row0 = rank * rows  # element-range shard of the global [world*rows, cols] array

    def data(rec):
        if rec["op"] not in ("VAR", "CONST"):
            return None
        shp = rec["shape"]
        off = row0 if (len(shp) == 2 and shp[0] == rows) else 0
        return materialise(rec["data"], shp, row_offset=off)

    g, outs = cg.build_from_spec(spec, device=local, data_fn=data)
    rep = g.optimise(outs)
    info = g.plan_memory(outs, 0)
    ws = torch.cuda.ExternalStream(g.work_stream(), device=torch.device("cuda", local))
    algo = configs.c2_algo_bytes(rows, cols)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        g.eval(outs, cg.EVAL_FULL)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    # keep the GPU under this same load for ~0.5 s before the timed region so the
    # sampled clocks are the clocks of the measured kernel (nvidia-smi samples every 100 ms)
    t_end = time.perf_counter() + 0.5
    while time.perf_counter() < t_end:
        for _ in range(20):
            g.eval(outs, cg.EVAL_FULL)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
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
    if world > 1:
        t = torch.tensor([ms, kernel_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kernel_ms = float(t[0]), float(t[1])
        dist.barrier()
    value = world * algo / (ms * 1e-3) / 1e9

    # e2e: through the public API with HOST buffers (pinned), copies inside the timed region
    e2e_steps = max(1, min(args.steps, 3))
    hx = torch.from_numpy(data(spec["nodes"][0])).pin_memory()
    hy = torch.from_numpy(data(spec["nodes"][1])).pin_memory()
    hout = torch.empty((rows, cols), dtype=torch.float32).pin_memory()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        g.assign(0, hx)
        g.assign(1, hy)
        g.eval(outs)
        g.read_into(outs[0], hout)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    e2e_val = world * algo / (e2e_ms * 1e-3) / 1e9

    secondary = None
    if not args.no_secondary:
        # the C2 line must survive a failure in the secondary configs (e.g. an NCCL
        # communicator that cannot be created on some box); a failure that every
        # rank sees identically (setup) keeps the ranks in step
        try:
            secondary = run_secondary(rank, world, local, max(5, args.steps))
        except Exception as exc:  # noqa: BLE001
            import traceback
            traceback.print_exc(file=sys.stderr)
            secondary = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if rank == 0:
        hbm, how = peaks()
        achieved = algo / (kernel_ms * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "c2_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            gbs, sample, _ = oracle_c2_rate(budget_s=args.cpu_budget)
            cpu = {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample}
        line = {
            "metric": "fused graph-eval HBM GB/s", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded splitmix64)",
            "config": {"workload": "C2: 20-op elementwise/broadcast chain (CSE+CF -> 17 ops, 1 fused kernel)",
                       "rows_per_gpu": rows, "cols": cols, "elements_per_gpu": rows * cols,
                       "algorithmic_bytes_per_step_per_gpu": algo, "parallelism": f"element-range x{world}",
                       "l2": "3 GiB moved per step >> 126 MB L2: no flush needed",
                       "eval": "CG_EVAL_FULL (no reuse of pre-computed nodes, P:385)",
                       "optimiser": rep, "plan": {k: info[k] for k in ("n_groups", "n_blocks", "pool_bytes",
                                                                       "unshared_bytes")}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_source": how,
                         "kernel_ms": kernel_ms},
            "clocks": clk,
            "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": 2 * rows * cols * 4,
                    "d2h_bytes_per_step": rows * cols * 4, "ms_per_step": e2e_ms},
            "gpu_launches": launches,
            "cpu_baseline": cpu,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- secondary workloads
def _time_region(ws, fn, iters):
    import torch
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(ws)
    for k in range(iters):
        fn(k)
    e.record(ws)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def run_secondary(rank, world, local, iters):
    """BASELINE.json's other metrics on the other configs: C1 full / incremental
    eval latency, C3 / C4 data-parallel training iterations per second (global
    batch fixed: 4096 / 8192, split over the ranks), C5 images/s with the plan's
    peak bytes vs the unshared (eager) allocation."""
    import torch

    from paper_1812_03770_b200 import cg
    from paper_1812_03770_b200.dist import dp_spec, make_graph, shard_range
    from workloads import configs
    from workloads.gen import materialise, retag

    out = {}
    dev = torch.device("cuda", local)

    def leaf(rec, off=0):
        if rec["op"] not in ("VAR", "CONST"):
            return None
        return materialise(rec["data"], rec["shape"], row_offset=off)

    # C1: Fig. 1 graph, full eval and incremental re-eval after cg_assign(x3)
    spec = configs.c1(1024)
    g, outs = cg.build_from_spec(spec, device=local, data_fn=leaf)
    g.plan_memory(outs, cg.PLAN_INCREMENTAL)
    ws = torch.cuda.ExternalStream(g.work_stream(), device=dev)
    x3 = [torch.from_numpy(materialise(retag(spec["nodes"][3]["data"], f"x3#{k}"), [1024])).to(dev) for k in range(2)]
    for _ in range(5):
        g.eval(outs, cg.EVAL_FULL)
    torch.cuda.synchronize()
    full_ms = _time_region(ws, lambda k: g.eval(outs, cg.EVAL_FULL), 200)

    def inc(k):
        g.assign(3, x3[k % 2])
        g.eval(outs)
    inc_ms = _time_region(ws, inc, 200)
    out["C1"] = {"metric": "eval latency", "unit": "us", "full_eval_us": full_ms * 1e3,
                 "incremental_eval_us (assign x3 + eval)": inc_ms * 1e3, "x2_evaluations": g.eval_count(2),
                 "x5_evaluations": g.eval_count(5)}
    g.destroy()

    # C3 / C4: data-parallel training, global batch split over ranks (strong scaling)
    for name, fn, gb in (("C3", configs.c3, 4096), ("C4", configs.c4, 8192)):
        spec = dp_spec(fn, gb, rank, world)
        start, count = shard_range(gb, rank, world)
        g = make_graph(local, world, rank)
        for rec in spec["nodes"]:
            data = leaf(rec)
            if rec["op"] in ("VAR", "CONST"):
                g.add_node(rec["op"], (), dims=rec["shape"], **({"data": data} if data is not None else {}))
            else:
                g.add_node(rec["op"], rec["preds"], **rec.get("attrs", {}))
        for u, v in spec["updates"]:
            g.add_update(u, v)
        outs = spec["outputs"]
        g.optimise(outs)
        info = g.plan_memory(outs, 0)
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
        for k in range(3):
            step(k)
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        ms = _max_over_ranks(_time_region(ws, step, iters), world)
        out[name] = {"metric": "train iters/s", "value": 1e3 / ms, "unit": "iters/s", "ms_per_iter": ms,
                     "global_batch": gb, "local_batch": count, "scaling": "strong",
                     "parallelism": f"dp{world}" + (" (NCCL AllReduce nodes)" if world > 1 else ""),
                     "plan_peak_bytes": info["pool_bytes"] + info["external_bytes"] + info["workspace_bytes"],
                     "unshared_bytes": info["unshared_bytes"] + info["external_bytes"]}
        g.destroy()

    # C5: InceptionV3 inference, 256 images per GPU (batch-sharded replicas)
    spec = configs.c5()
    g, outs = cg.build_from_spec(spec, device=local, data_fn=leaf)
    g.optimise(outs)
    info = g.plan_memory(outs, 0)
    ws = torch.cuda.ExternalStream(g.work_stream(), device=dev)
    for _ in range(2):
        g.eval(outs, cg.EVAL_FULL)
    torch.cuda.synchronize()
    ms = _max_over_ranks(_time_region(ws, lambda k: g.eval(outs, cg.EVAL_FULL), max(2, iters // 4)), world)
    peak = info["pool_bytes"] + info["external_bytes"] + info["workspace_bytes"]
    unshared = info["unshared_bytes"] + info["external_bytes"]
    out["C5"] = {"metric": "images/s", "value": world * 256 / (ms * 1e-3), "unit": "images/s", "ms_per_eval": ms,
                 "batch_per_gpu": 256, "scaling": "weak", "plan_peak_bytes": peak, "unshared_bytes": unshared,
                 "peak_vs_unshared": peak / unshared, "n_groups": info["n_groups"], "n_blocks": info["n_blocks"]}
    g.destroy()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="C2 only (skip the C1/C3/C4/C5 lines)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == "C2":
        run_c2(args)
    else:
        raise SystemExit(f"config {args.config} not wired into bench.py yet")


if __name__ == "__main__":
    main()
