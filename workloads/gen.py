"""Seeded, counter-based synthetic input generator (SURVEY.md §8(d) "Data generator").

This module is INPUT GENERATION ONLY.  It holds none of the method's
arithmetic (no graph evaluation, rewriting or planning) and is the one
module that both the oracle (``oracle/``) and the CUDA path's harness
(``tests/``, ``bench.py``) import.  Values are indexable by flat row-major
element index, so a shard or a sampled row set regenerates exactly the bits
of the full tensor.

    splitmix64(z): z += 0x9E3779B97F4A7C15
                   z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
                   z = (z ^ (z >> 27)) * 0x94D049BB133111EB
                   return z ^ (z >> 31)                       (all mod 2^64)
    H(seed, tag)  = splitmix64(seed ^ FNV-1a-64(tag))
    u(seed,tag,i) = (splitmix64(H(seed, tag) + i) >> 40) * 2^-24   in [0, 1), exact in fp32
    value         = lo + (hi - lo) * u    computed in f64, rounded to fp32
    label(row)    = floor(classes * u(seed, tag, row))  -> one-hot row
"""
from __future__ import annotations

import concurrent.futures as _cf
import os

import numpy as np

SEED = 1812

_M64 = (1 << 64) - 1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def fnv1a64(tag: str) -> int:
    h = 0xCBF29CE484222325
    for b in tag.encode("utf-8"):
        h ^= b
        h = (h * 0x100000001B3) & _M64
    return h


def splitmix64_int(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream_key(seed: int, tag: str) -> int:
    return splitmix64_int((seed ^ fnv1a64(tag)) & _M64)


def _splitmix64_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        return z ^ (z >> np.uint64(31))


def _u_of(key: int, idx: np.ndarray) -> np.ndarray:
    """u for flat indices ``idx`` (uint64 array) as float64 in [0, 1)."""
    with np.errstate(over="ignore"):
        z = idx.astype(np.uint64) + np.uint64(key)
    return (_splitmix64_np(z) >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


_CHUNK = 1 << 22


def uniform_flat(seed: int, tag: str, lo: float, hi: float, idx: np.ndarray) -> np.ndarray:
    """fp32 values at the given flat element indices."""
    key = stream_key(seed, tag)
    idx = np.asarray(idx, dtype=np.uint64).ravel()
    out = np.empty(idx.shape[0], dtype=np.float32)
    lo = float(lo)
    span = float(hi) - float(lo)

    def work(s):
        e = min(s + _CHUNK, idx.shape[0])
        out[s:e] = (lo + span * _u_of(key, idx[s:e])).astype(np.float32)

    starts = range(0, idx.shape[0], _CHUNK)
    if idx.shape[0] > 4 * _CHUNK:
        with _cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            list(ex.map(work, starts))
    else:
        for s in starts:
            work(s)
    return out


def uniform_range(seed: int, tag: str, lo: float, hi: float, start: int, count: int) -> np.ndarray:
    """fp32 values at flat indices [start, start + count) without building an index array per element."""
    key = stream_key(seed, tag)
    out = np.empty(count, dtype=np.float32)
    lo = float(lo)
    span = float(hi) - float(lo)

    def work(s):
        e = min(s + _CHUNK, count)
        idx = np.arange(start + s, start + e, dtype=np.uint64)
        out[s:e] = (lo + span * _u_of(key, idx)).astype(np.float32)

    starts = range(0, count, _CHUNK)
    if count > 4 * _CHUNK:
        with _cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            list(ex.map(work, starts))
    else:
        for s in starts:
            work(s)
    return out


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= int(d)
    return n


def materialise(data: dict, shape, seed: int = SEED, rows=None, row_offset: int = 0) -> np.ndarray:
    """Build the fp32 tensor a data spec describes.

    ``data`` kinds (the graph-spec format of workloads/configs.py):
      {"kind": "uniform", "tag": t, "lo": a, "hi": b}
      {"kind": "onehot",  "tag": t, "classes": k}     (shape [B, k]; row r uses u(seed,t,r))
      {"kind": "literal", "values": [...]}            (row-major, len == numel)
      {"kind": "zeros"} / {"kind": "full", "value": v}
    ``rows``: optional sequence of leading-axis indices to generate (sampling);
    ``row_offset``: the leading-axis index of local row 0 in the global tensor
    (element-range / batch sharding).  Both refer to the GLOBAL tensor, so a
    shard or a sample reproduces the global tensor's bits.
    """
    shape = tuple(int(d) for d in shape)
    kind = data["kind"]
    if rows is not None:
        rows = np.asarray(rows, dtype=np.int64)
        out_shape = (rows.shape[0],) + shape[1:]
    else:
        out_shape = shape
    rowsize = _numel(shape[1:]) if len(shape) >= 1 else 1

    if kind == "uniform":
        if rows is None:
            flat = uniform_range(seed, data["tag"], data["lo"], data["hi"],
                                 row_offset * rowsize, _numel(shape))
        else:
            g = (rows + row_offset)[:, None] * rowsize + np.arange(rowsize, dtype=np.int64)[None, :]
            flat = uniform_flat(seed, data["tag"], data["lo"], data["hi"], g.ravel())
        return flat.reshape(out_shape)
    if kind == "onehot":
        k = int(data["classes"])
        assert len(shape) == 2 and shape[1] == k, "onehot wants shape [B, classes]"
        r = (rows if rows is not None else np.arange(shape[0], dtype=np.int64)) + row_offset
        u = _u_of(stream_key(seed, data["tag"]), r.astype(np.uint64))
        lab = np.floor(k * u).astype(np.int64)
        out = np.zeros(out_shape, dtype=np.float32)
        out[np.arange(out_shape[0]), lab] = 1.0
        return out
    if kind == "literal":
        vals = np.asarray(data["values"], dtype=np.float32).reshape(shape)
        if rows is not None:
            vals = vals[rows]
        return np.array(vals, order="C")
    if kind == "zeros":
        return np.zeros(out_shape, dtype=np.float32)
    if kind == "full":
        return np.full(out_shape, np.float32(data["value"]), dtype=np.float32)
    raise ValueError(f"unknown data kind {kind!r}")


def retag(data: dict, tag: str) -> dict:
    """Same distribution, another counter stream (e.g. per-iteration batches "X@3")."""
    d = dict(data)
    if "tag" in d:
        d["tag"] = tag
    return d
