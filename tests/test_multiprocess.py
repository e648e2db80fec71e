"""Multi-process (world size 2, gloo, CPU) tests of the data-parallel host logic
(DESIGN.md §9).  No GPU: the decomposition the GPU path relies on
is checked with the oracle and the host-only planner, rank by rank."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.eager import evaluate, leaf_values
from oracle.graph import from_spec
from paper_1812_03770_b200 import cg
from paper_1812_03770_b200.dist import broadcast_nccl_id, dp_spec, shard_range
from workloads import configs
from workloads.gen import materialise

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(fn, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(r, port, fn, args, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = {}
    for _ in procs:
        r, ok, payload = q.get(timeout=600)
        results[r] = (ok, payload)
    for p in procs:
        p.join(timeout=60)
    for r, (ok, payload) in sorted(results.items()):
        assert ok, f"rank {r}: {payload}"
    return {r: payload for r, (_, payload) in results.items()}


def _entry(rank, port, fn, args, q):
    import traceback
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        out = fn(rank, *args)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, True, out))
    except Exception:  # pragma: no cover - reported by the parent
        q.put((rank, False, traceback.format_exc()))


def test_shard_range_partitions():
    for total in (0, 1, 7, 4096, 8192, 262144):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                s, c = shard_range(total, r, world)
                covered.extend(range(s, s + c))
            assert covered == list(range(total))


# ---------------------------------------------------------------- NCCL id exchange
def _uid_rank(rank):
    fake = bytes((i * 7 + 3) % 256 for i in range(128))
    uid = broadcast_nccl_id(make_id=lambda: fake)
    return uid.hex()


def test_nccl_id_broadcast():
    res = _run(_uid_rank)
    assert res[0] == res[1] == bytes((i * 7 + 3) % 256 for i in range(128)).hex()


# ---------------------------------------------------------------- identical plans on every rank
def _plan_rank(rank):
    spec = dp_spec(configs.c3, 4096, rank, WORLD)
    g, _ = cg.build_from_spec(spec, device=-1, rank=rank, world=WORLD,
                              data_fn=lambda r: materialise(r["data"], r["shape"]) if r["op"] == "CONST" else None)
    g.optimise(spec["outputs"])
    g.plan_memory(spec["outputs"])
    plan = g.dump_json(cg.DUMP_PLAN)
    allp = [None] * WORLD
    dist.all_gather_object(allp, plan)
    return allp[0] == allp[1]


def test_dp_plans_identical_across_ranks():
    """Every rank builds the same graph with local-batch shapes, so
    the host compiler produces byte-identical plans: the NCCL calls captured in
    each rank's CUDA graph line up."""
    res = _run(_plan_rank)
    assert res[0] and res[1]


# ---------------------------------------------------------------- DP gradient = full-batch gradient
def _grad_rank(rank, batch):
    """Oracle on this rank's batch shard; sum the local gradients over ranks with
    gloo (what ALLREDUCE_SUM does on the GPU) and return them."""
    spec = dp_spec(configs.c3, batch, rank, WORLD, widths=(784, 64, 32, 10))
    start, _ = shard_range(batch, rank, WORLD)
    og, _ = from_spec(spec)
    over = {}
    for n in og.nodes:
        if n.op == "VAR" and n.name in ("X", "Y"):
            over[n.id] = materialise(n.data, n.shape, row_offset=start)
    vals = evaluate(og, leaf_values(og, over), dtype=np.float64)
    grads = {}
    for n in og.nodes:
        if n.op == "ALLREDUCE_SUM":
            t = torch.from_numpy(np.ascontiguousarray(vals[n.preds[0]], dtype=np.float64))
            dist.all_reduce(t)
            grads[n.id] = t.numpy()
    return grads


def test_dp_gradient_sum_equals_full_batch():
    """c10: with the loss scaled by 1/B_global, the sum over ranks of the local
    gradients equals the single-process full-batch gradient."""
    batch = 64
    res = _run(_grad_rank, batch)
    spec = configs.c3(batch=batch, widths=(784, 64, 32, 10))
    og, _ = from_spec(spec)
    vals = evaluate(og, leaf_values(og), dtype=np.float64)
    full = {n.id: vals[n.preds[0]] for n in og.nodes if n.op == "ALLREDUCE_SUM"}
    assert set(full) == set(res[0])
    for i, want in full.items():
        for r in range(WORLD):
            np.testing.assert_allclose(res[r][i], want, rtol=1e-9, atol=1e-12)


# ---------------------------------------------------------------- element-range sharding (no collective)
def _c2_rank(rank, rows, cols):
    start, count = shard_range(rows, rank, WORLD)
    spec = configs.c2(rows=count, cols=cols)
    og, oo = from_spec(spec)
    over = {}
    for n in og.nodes:
        if n.op in ("VAR", "CONST") and len(n.shape) == 2 and n.shape[0] == count:
            over[n.id] = materialise(n.data, n.shape, row_offset=start)
    vals = leaf_values(og)
    vals.update(over)  # this rank's row range of the [rows, ...] Vars and Consts
    return evaluate(og, vals)[oo[0]]


def test_c2_element_range_shards_concatenate_to_full():
    rows, cols = 96, 64
    res = _run(_c2_rank, rows, cols)
    og, oo = from_spec(configs.c2(rows=rows, cols=cols))
    full = evaluate(og, leaf_values(og))[oo[0]]
    assert np.array_equal(np.concatenate([res[0], res[1]], axis=0), full)


def _host_data(rec):
    return materialise(rec["data"], rec["shape"]) if rec["op"] == "CONST" else None


class _FakeGraph:
    """Stands in for a planned cg.Graph on CPU: a per-rank handle, records connect."""

    def __init__(self, rank):
        self.handle = bytes([rank + 1]) * 64 + bytes([0xA0 + rank]) * 64
        self.connected = None

    def coll_handle(self):
        return self.handle

    def coll_connect(self, handles):
        self.connected = list(handles)


def _fused_connect(rank):
    from paper_1812_03770_b200.dist import connect_fused
    g = _FakeGraph(rank)
    connect_fused(g)
    return [h.hex() for h in g.connected]


def test_fused_coll_handle_exchange():
    """connect_fused (CG_PLAN_FUSED_COLL, f3): every rank receives every rank's
    128-byte peer-memory handle, in rank order, identically."""
    res = _run(_fused_connect)
    want = [(bytes([r + 1]) * 64 + bytes([0xA0 + r]) * 64).hex() for r in range(WORLD)]
    for r in range(WORLD):
        assert res[r] == want


def test_fused_coll_flag_host_only_plan():
    """The flag is an executor choice: a host-only plan with it equals the plain plan."""
    spec = configs.c3(batch=64, widths=(784, 32, 10))
    dumps = []
    for flags in (0, cg.PLAN_FUSED_COLL):
        g, outs = cg.build_from_spec(spec, device=-1, data_fn=_host_data)
        g.optimise(outs)
        g.plan_memory(outs, flags)
        dumps.append(g.dump_json(cg.DUMP_PLAN))
        g.destroy()
    assert dumps[0] == dumps[1]
