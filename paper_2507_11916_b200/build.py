"""Builds the in-tree CUDA library for sm_100a (no torch JIT cache)."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libbida_gpu.so")
SOURCES = ["bida_gpu.cu", "mlp.cu", "pdb_build.cu", "walks.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-I" + os.path.join(ROOT, "include"),
]


def _stale(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "bida_gpu.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


OUT_TRACE = os.path.join(HERE, "_lib", "libbida_gpu_trace.so")


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace=True: the diagnostic variant with the clock64 kernel timeline
    compiled in (tests/trace_mlp.py; loaded when BIDA_GPU_TRACE=1).  Sources
    compile in parallel, then link into one shared library."""
    out = OUT_TRACE if trace else OUT
    if not force and not _stale(out):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objdir = os.path.join(HERE, "_lib", "obj_trace" if trace else "obj")
    os.makedirs(objdir, exist_ok=True)
    extra = (["-DBIDA_MLP_TRACE=1"] if trace else []) + (["-Xptxas=-v"] if verbose else [])

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        subprocess.run([NVCC, *FLAGS, *extra, "-c", "-o", obj, os.path.join(CSRC, src)], check=True)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = out + ".tmp"
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
