"""Data-parallel plumbing for the evaluator (one process per GPU) [P:26, P:42].

The paper claims "natural support for parallel and distributed computing"
 and notes that vertices "might be computed on different machines"
without a concrete scheme; SURVEY §8(e) fixes two:

* element-range sharding of pure elementwise/broadcast graphs (C2): rank r owns
  rows [r*R/P, (r+1)*R/P) of the leading axis; no collective on the data path;
* batch data parallelism of training graphs (C3, C4): rank r owns samples
  [r*B/P, (r+1)*B/P); the graph carries ALLREDUCE_SUM nodes on the gradients
  (ncclAllReduce on the graph's stream, inside the captured CUDA graph) and the
  loss is scaled by 1/B_global, so the summed gradient is the global-batch mean.

torch.distributed is used only to exchange the 128-byte NCCL unique id (or the
128-byte peer-memory handles of the fused collectives, CG_PLAN_FUSED_COLL) and for
barriers / max-over-ranks timing; the collective itself runs inside libcg.so.
"""
from __future__ import annotations

import os

from . import cg


def env_rank_world():
    """(rank, world, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block partition of ``total`` leading-axis items: (start, count).
    Blocks differ in size by at most one; every item is owned by exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def broadcast_nccl_id(make_id=None) -> bytes:
    """Rank 0 creates the NCCL unique id (cg_nccl_unique_id unless ``make_id`` is
    given) and every rank receives it over the torch process group."""
    import torch.distributed as dist

    obj = [None]
    if dist.get_rank() == 0:
        obj[0] = bytes(make_id() if make_id else cg.nccl_unique_id())
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("NCCL unique id must be 128 bytes")
    return bytes(uid)


def make_graph(device: int, world: int | None = None, rank: int | None = None, nccl_id: bytes | None = None,
               fused: bool = False):
    """cg.Graph on ``device``; with world > 1 it owns an NCCL communicator for its
    ALLREDUCE_SUM nodes (the unique id is broadcast if not supplied) -- or, with
    ``fused``, none: the graph is then planned with cg.PLAN_FUSED_COLL and
    connected with connect_fused()."""
    import torch.distributed as dist

    if world is None:
        world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    if world <= 1:
        return cg.Graph(device)
    if rank is None:
        rank = dist.get_rank()
    if fused:
        return cg.Graph(device, rank=rank, world=world, nccl_id=None)
    if nccl_id is None:
        nccl_id = broadcast_nccl_id()
    return cg.Graph(device, rank=rank, world=world, nccl_id=nccl_id)


def gather_handles(handle: bytes) -> list:
    """Every rank's 128-byte peer-memory handle, in rank order (all_gather_object
    over the torch process group; world 1: just this one)."""
    import torch.distributed as dist

    if len(handle) != 128:
        raise ValueError("peer-memory handle must be 128 bytes")
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [bytes(handle)]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, bytes(handle))
    if any(not isinstance(h, (bytes, bytearray)) or len(h) != 128 for h in out):
        raise RuntimeError("a rank sent a malformed peer-memory handle")
    return [bytes(h) for h in out]


def connect_fused(g) -> None:
    """After g.plan_memory(..., cg.PLAN_FUSED_COLL): exchange the peer-memory handles
    and map every rank's pool and flag words (cg_coll_connect)."""
    g.coll_connect(gather_handles(g.coll_handle()))


def dp_spec(config_fn, global_batch: int, rank: int, world: int, **kw) -> dict:
    """Per-rank training spec of a data-parallel run: local batch B/P (block
    partition), loss scaled by 1/B_global, gradients through ALLREDUCE_SUM."""
    _, count = shard_range(global_batch, rank, world)
    return config_fn(batch=count, batch_global=global_batch, **kw)
