"""Builds libautooverlap.so in-tree with nvcc for sm_100a only.

`python -m paper_2601_20595_b200.build` (or __graft_entry__.build()).  The library is
compiled with `-gencode arch=compute_100a,code=sm_100a` (never `-arch=sm_100a`, which also
emits a generic compute_100 PTX pass that rejects tcgen05) and -lineinfo so
ncu's source page maps to the kernels.  No CUDA device is needed to build.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libautooverlap.so")
SOURCES = ["planner.cpp", "runtime.cpp", "fused.cu", "a2a.cu", "attn.cu", "e4.cu"]
HEADERS = ["planner.h", "kernel_args.h", "ptx.cuh", "transfer.cuh"]


def nvcc_path():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_rebuild():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "autooverlap.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = True) -> str:
    """Compiles every translation unit in parallel (one nvcc per file), then links."""
    if not force and not needs_rebuild():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    nvcc = nvcc_path()
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    base = [nvcc, "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
            "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-I", INCLUDE, "-I", CSRC,
            "-Xptxas", "-v" if os.environ.get("AO_PTXAS_VERBOSE") else "-O3"]
    extra = os.environ.get("AO_NVCC_FLAGS", "").split()

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = base + extra + ["-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.stderr:
            sys.stderr.write(r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp"] + objs
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
