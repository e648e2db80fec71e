"""Python binding of the C ABI in include/cg.h (argument marshalling only).

Every function here forwards to libcg.so through ctypes under the C name it
mirrors (cg_create, cg_add_node, cg_add_update, cg_optimise, cg_plan_memory,
cg_assign, cg_eval, cg_read, cg_destroy, ...).  No step of the evaluation
runs in Python; if the shared library is missing the import fails loudly —
there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcg.so")

OPS = ["VAR", "CONST", "ADD", "SUB", "MUL", "DIV", "POW", "MAX2", "MIN2", "RELU_GRAD", "FMA",
       "NEG", "ABS", "SQRT", "EXP", "LOG", "SIN", "COS", "TANH", "RELU", "SUM", "MAX", "DOT",
       "CONV2D", "CONV2D_BWD_INPUT", "CONV2D_BWD_KERNEL", "MAXPOOL2D", "MAXPOOL2D_BWD", "AVGPOOL2D",
       "CONCAT", "RESHAPE", "ALLREDUCE_SUM", "FUSED_ADAGRAD"]
OP_CODE = {n: i for i, n in enumerate(OPS)}

STATUS = {0: "CG_OK", -1: "CG_E_ARITY", -2: "CG_E_BAD_NODE", -3: "CG_E_SHAPE", -4: "CG_E_NOT_VAR",
          -5: "CG_E_DUP_UPDATE", -6: "CG_E_UPDATE_SHAPE", -7: "CG_E_NOT_PLANNED", -8: "CG_E_SIZE",
          -9: "CG_E_STATE", -10: "CG_E_CUDA", -11: "CG_E_NCCL", -12: "CG_E_NVRTC", -13: "CG_E_OOM",
          -14: "CG_E_ARG", -15: "CG_E_NO_DEVICE"}

PLAN_INCREMENTAL = 1
PLAN_NO_FUSION = 2
PLAN_FUSED_COLL = 4
EVAL_NO_UPDATE = 1
EVAL_FULL = 2
EVAL_SYNC = 4
RW_IDENTITY = 1
RW_FMA = 2
RW_ADAGRAD = 4
RW_ALL = 7
DUMP_GRAPH = 0
DUMP_PLAN = 1

# names exported by include/cg.h (tests check the library exports every one)
ABI_SYMBOLS = ["cg_create", "cg_add_node", "cg_add_update", "cg_optimise", "cg_plan_memory", "cg_assign",
               "cg_eval", "cg_read", "cg_destroy", "cg_last_error", "cg_nccl_unique_id", "cg_dump_json",
               "cg_eval_count", "cg_node_shape", "cg_launch_count", "cg_set_rewrites", "cg_coll_handle",
               "cg_coll_connect"]


class cg_attr(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("dims", ctypes.c_int64 * 8), ("host_data", ctypes.c_void_p),
                ("a0", ctypes.c_int32), ("a1", ctypes.c_int32), ("ta", ctypes.c_int32), ("tb", ctypes.c_int32),
                ("sh", ctypes.c_int32), ("sw", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("kh", ctypes.c_int32), ("kw", ctypes.c_int32), ("h", ctypes.c_int32), ("w", ctypes.c_int32),
                ("axis", ctypes.c_int32)]


class cg_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p)]


class cg_report(ctypes.Structure):
    _fields_ = [("cse_merged", ctypes.c_int32), ("cf_folded", ctypes.c_int32), ("dce_removed", ctypes.c_int32),
                ("rw_identity", ctypes.c_int32), ("rw_zeroed", ctypes.c_int32), ("rw_fma", ctypes.c_int32),
                ("rw_adagrad", ctypes.c_int32)]


class cg_plan_info(ctypes.Structure):
    _fields_ = [("n_groups", ctypes.c_int32), ("n_blocks", ctypes.c_int32), ("n_kernels", ctypes.c_int32),
                ("n_fused", ctypes.c_int32), ("pool_bytes", ctypes.c_uint64), ("plan_bytes", ctypes.c_uint64),
                ("external_bytes", ctypes.c_uint64), ("workspace_bytes", ctypes.c_uint64),
                ("unshared_bytes", ctypes.c_uint64)]


_lib = None


def lib():
    """Load libcg.so (raises if it was not built: the CUDA path has no substitute)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_1812_03770_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, U32, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
        sig = {
            "cg_create": (P, [ctypes.c_int, P, P]),
            "cg_add_node": (I32, [P, ctypes.c_int, P, I32, P]),
            "cg_add_update": (ctypes.c_int, [P, I32, I32]),
            "cg_optimise": (ctypes.c_int, [P, P, I32, P]),
            "cg_set_rewrites": (ctypes.c_int, [P, U32]),
            "cg_plan_memory": (ctypes.c_int, [P, P, I32, U32, P]),
            "cg_assign": (ctypes.c_int, [P, I32, P, SZ, ctypes.c_int]),
            "cg_eval": (ctypes.c_int, [P, P, I32, P, U32]),
            "cg_read": (ctypes.c_int, [P, I32, P, SZ]),
            "cg_destroy": (None, [P]),
            "cg_last_error": (ctypes.c_char_p, [P]),
            "cg_nccl_unique_id": (ctypes.c_int, [P]),
            "cg_dump_json": (I64, [P, ctypes.c_int, P, SZ]),
            "cg_eval_count": (I64, [P, I32]),
            "cg_node_shape": (I32, [P, I32, P]),
            "cg_launch_count": (I64, [P]),
            "cg_coll_handle": (ctypes.c_int, [P, P, SZ]),
            "cg_coll_connect": (ctypes.c_int, [P, P, I32]),
            "cgx_collective_schedule": (I32, [I32, P, P, P, P, P, P, P, P, P]),
            "cgx_coll_batches": (I64, [P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class CGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = STATUS.get(code, code)


def _ids(xs):
    arr = (ctypes.c_int32 * max(1, len(xs)))(*[int(x) for x in xs])
    return arr


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().cg_nccl_unique_id(buf)
    if rc < 0:
        raise CGError(rc, lib().cg_last_error(None).decode())
    return buf.raw


def collective_schedule(rd, wr, uses_ws, is_coll, active=None):
    """cgx_collective_schedule on synthetic access sets (lists of block-id lists per
    group).  Returns a list of steps (lists of group ids) in issue order."""
    ng = len(rd)

    def csr(sets):
        ptr = np.zeros(ng + 1, np.int32)
        for i, s_ in enumerate(sets):
            ptr[i + 1] = ptr[i] + len(s_)
        idx = np.array([b for s_ in sets for b in s_] or [0], np.int32)
        return ptr, idx
    rp, ri = csr(rd)
    wp, wi = csr(wr)
    ws = np.asarray(uses_ws, np.uint8)
    co = np.asarray(is_coll, np.uint8)
    act = None if active is None else np.asarray(active, np.uint8)
    order = np.zeros(max(ng, 1), np.int32)
    step = np.zeros(max(ng, 1), np.int32)
    n = lib().cgx_collective_schedule(ng, None if act is None else act.ctypes.data, rp.ctypes.data, ri.ctypes.data,
                                      wp.ctypes.data, wi.ctypes.data, ws.ctypes.data, co.ctypes.data,
                                      order.ctypes.data, step.ctypes.data)
    if n < 0:
        raise CGError(n, "cgx_collective_schedule")
    steps = []
    for k in range(n):
        if k == 0 or step[k] != step[k - 1]:
            steps.append([])
        steps[-1].append(int(order[k]))
    return steps


class Graph:
    """One cg_graph.  device=-1: host-only planning mode (structure only)."""

    def __init__(self, device: int = 0, stream=None, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        L = lib()
        self._keep = []
        dist = None
        if world > 1 or nccl_id:  # world == 1 with an id: a 1-rank NCCL communicator
            self._uid = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
            dist = cg_dist(rank, world, ctypes.cast(self._uid, ctypes.c_void_p) if self._uid else None)
        if stream is None and device >= 0:
            try:
                import torch
                stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:  # pragma: no cover
                stream = 0
        self.h = L.cg_create(int(device), ctypes.c_void_p(stream or 0), ctypes.byref(dist) if dist else None)
        if not self.h:
            raise CGError(-10, L.cg_last_error(None).decode())
        self.device = device
        self.shapes = {}

    # ---- errors
    def _check(self, rc):
        if rc < 0:
            raise CGError(rc, lib().cg_last_error(self.h).decode())
        return rc

    # ---- build
    def add_node(self, op: str, inputs=(), **attrs) -> int:
        a = cg_attr()
        data = None
        for k, v in attrs.items():
            if k == "dims":
                a.ndim = len(v)
                for i, d in enumerate(v):
                    a.dims[i] = int(d)
            elif k == "data":
                data = np.ascontiguousarray(np.asarray(v, dtype=np.float32))
                self._keep.append(data)
                a.host_data = data.ctypes.data
            else:
                setattr(a, k, int(v))
        if op in ("VAR", "CONST"):
            shape = attrs.get("dims", ())
            if data is not None and data.size != int(np.prod(shape, dtype=np.int64)):
                raise ValueError("data size does not match shape")
        rc = lib().cg_add_node(self.h, OP_CODE[op], _ids(inputs), len(inputs), ctypes.byref(a))
        self._check(rc)
        if op in ("VAR", "CONST"):
            self._keep.clear()  # data copied by the library
        return rc

    def var(self, shape, init=None) -> int:
        kw = {"dims": list(shape)}
        if init is not None:
            kw["data"] = init
        return self.add_node("VAR", (), **kw)

    def const(self, value, shape=None) -> int:
        value = np.asarray(value, dtype=np.float32)
        return self.add_node("CONST", (), dims=list(shape if shape is not None else value.shape), data=value)

    def add_update(self, u: int, var: int):
        self._check(lib().cg_add_update(self.h, int(u), int(var)))

    def optimise(self, outputs) -> dict:
        r = cg_report()
        self._check(lib().cg_optimise(self.h, _ids(outputs), len(outputs), ctypes.byref(r)))
        return {f: getattr(r, f) for f, _ in cg_report._fields_}

    def set_rewrites(self, flags: int = 7):
        """cg_set_rewrites: the paper's pattern rewrites for the next optimise (RW_* flags)."""
        self._check(lib().cg_set_rewrites(self.h, int(flags)))

    def plan_memory(self, outputs, flags: int = 0) -> dict:
        info = cg_plan_info()
        self._check(lib().cg_plan_memory(self.h, _ids(outputs), len(outputs), int(flags), ctypes.byref(info)))
        return {f: getattr(info, f) for f, _ in cg_plan_info._fields_}

    # ---- fused collectives (CG_PLAN_FUSED_COLL)
    def view_stats(self) -> dict:
        """Zero-copy CONCAT slices (R14): written directly by their producer / via scratch."""
        f = lib().cgx_view_stats
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        out = (ctypes.c_int64 * 2)()
        self._check(f(self.h, out))
        return {"direct": int(out[0]), "copied": int(out[1])}

    def coll_handle(self) -> bytes:
        """cg_coll_handle: this rank's 128-byte peer-memory handle (pool + flag words)."""
        buf = ctypes.create_string_buffer(128)
        self._check(lib().cg_coll_handle(self.h, buf, 128))
        return buf.raw

    def coll_connect(self, handles):
        """cg_coll_connect: ``handles`` = every rank's coll_handle() in rank order."""
        blob = b"".join(bytes(h) for h in handles)
        self._check(lib().cg_coll_connect(self.h, blob, len(handles)))

    # ---- run
    def assign(self, var: int, value):
        """value: numpy array (host copy) or a CUDA torch tensor (device copy)."""
        if hasattr(value, "data_ptr") and getattr(value, "is_cuda", False):
            assert value.is_contiguous()
            self._check(lib().cg_assign(self.h, int(var), ctypes.c_void_p(value.data_ptr()),
                                        value.numel() * value.element_size(), 1))
        elif hasattr(value, "data_ptr"):  # pinned / CPU torch tensor
            # A PINNED source is copied asynchronously on the graph's stream (stream order
            # puts it before the next eval): the caller must not refill the buffer until
            # that eval (or a read / synchronize) has returned.  Pageable memory is staged
            # by the driver before cg_assign returns and may be reused at once.
            assert value.is_contiguous()
            self._check(lib().cg_assign(self.h, int(var), ctypes.c_void_p(value.data_ptr()),
                                        value.numel() * value.element_size(), 0))
        else:
            arr = np.ascontiguousarray(np.asarray(value, dtype=np.float32))
            self._check(lib().cg_assign(self.h, int(var), arr.ctypes.data, arr.nbytes, 0))

    def eval(self, outputs, flags: int = 0):
        ptrs = (ctypes.c_void_p * max(1, len(outputs)))()
        self._check(lib().cg_eval(self.h, _ids(outputs), len(outputs), ptrs, int(flags)))
        return [ptrs[i] for i in range(len(outputs))]

    def shape(self, node: int):
        dims = (ctypes.c_int64 * 8)()
        r = self._check(lib().cg_node_shape(self.h, int(node), dims))
        return tuple(dims[i] for i in range(r))

    def read(self, node: int) -> np.ndarray:
        shp = self.shape(node)
        out = np.empty(shp, dtype=np.float32)
        self._check(lib().cg_read(self.h, int(node), out.ctypes.data, out.nbytes))
        return out

    def read_into(self, node: int, host_tensor):
        """D2H of a node into a (pinned) torch CPU tensor."""
        self._check(lib().cg_read(self.h, int(node), ctypes.c_void_p(host_tensor.data_ptr()),
                                  host_tensor.numel() * 4))

    def view(self, ptr: int, shape):
        """Zero-copy torch view of a borrowed device pointer returned by eval()."""
        import torch

        class _Arr:
            pass
        a = _Arr()
        a.__cuda_array_interface__ = {"shape": tuple(int(d) for d in shape), "typestr": "<f4",
                                      "data": (int(ptr), False), "version": 2, "strides": None}
        return torch.as_tensor(a, device=f"cuda:{self.device}")

    # ---- introspection
    def dump_json(self, what: int) -> str:
        n = self._check(lib().cg_dump_json(self.h, what, None, 0))
        buf = ctypes.create_string_buffer(n + 1)
        self._check(lib().cg_dump_json(self.h, what, buf, n + 1))
        return buf.value.decode()

    def eval_count(self, node: int) -> int:
        return self._check(lib().cg_eval_count(self.h, int(node)))

    def launch_count(self) -> int:
        return self._check(lib().cg_launch_count(self.h))

    def coll_batches(self) -> int:
        """Collective batches (one ncclGroupStart/End each) issued so far."""
        return self._check(lib().cgx_coll_batches(self.h))

    def work_stream(self) -> int:
        """cudaStream_t (as int) that every kernel of this graph is launched on."""
        f = lib().cgx_work_stream
        f.restype = ctypes.c_void_p
        f.argtypes = [ctypes.c_void_p]
        return f(self.h) or 0

    def kernel_source(self, gi: int, num_sms: int = 148) -> str:
        f = lib().cgx_kernel_source
        f.restype = ctypes.c_int64
        f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
        n = f(self.h, gi, num_sms, None, 0)
        buf = ctypes.create_string_buffer(int(n) + 1)
        f(self.h, gi, num_sms, buf, n + 1)
        return buf.value.decode()

    def destroy(self):
        if getattr(self, "h", None):
            lib().cg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def build_from_spec(spec: dict, device: int = 0, data_fn=None, **kw):
    """Marshal a workloads graph spec into cg_add_node / cg_add_update calls.

    ``data_fn(record) -> np.ndarray`` supplies leaf data (the harness passes the
    seeded generator); VARs without data start at zero.  Returns (Graph, outputs)."""
    g = Graph(device, **kw)
    for rec in spec["nodes"]:
        op = rec["op"]
        if op in ("VAR", "CONST"):
            data = data_fn(rec) if data_fn is not None else None
            if op == "CONST" and data is None:
                raise ValueError(f"CONST {rec.get('name')} needs data")
            i = g.add_node(op, (), dims=rec["shape"], **({"data": data} if data is not None else {}))
        else:
            i = g.add_node(op, rec["preds"], **rec.get("attrs", {}))
        assert i == rec["id"]
    for u, v in spec.get("updates", []):
        g.add_update(u, v)
    return g, list(spec.get("outputs", []))
