"""Build libcg.so in-tree: nvcc for sm_100a, static cudart, NVRTC for generated kernels.

    python -m paper_1812_03770_b200.build          (or __graft_entry__.build())
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcg.so")
SOURCES = ["host.cpp", "codegen.cpp", "schedule.cpp", "kernels.cu", "dot_tc.cu", "dot_small.cu", "conv_small.cu", "conv_img_tc.cu", "coll.cu", "engine.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newest_source_mtime():
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    paths.append(os.path.join(HERE, "..", "include", "cg.h"))
    return max(os.path.getmtime(p) for p in paths)


def needs_build() -> bool:
    return not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest_source_mtime()


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(CSRC, "build", src + ".o")
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        extra = os.environ.get("CG_EXTRA_NVCC_FLAGS", "").split()  # measurement builds (e.g. -DCG_SB_TIMING)
        cmd = [NVCC, "-std=c++17", "-O3", "-lineinfo", "-diag-suppress=177", *extra, "-Xcompiler", "-fPIC,-O3", *ARCH,
               "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        cmds.append(cmd)
        objs.append(obj)
    # translation units compile independently: one nvcc per source, in parallel
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-shared", *ARCH, "-cudart", "static", *objs, "-o", tmp, "-lnvrtc", "-ldl",
           "-L/usr/local/cuda/lib64", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
