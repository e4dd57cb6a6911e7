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


STAMP = LIB + ".stamp"


def _source_digest():
    """sha256 over the sources, headers and extra nvcc flags the library is built from."""
    import hashlib
    h = hashlib.sha256(os.environ.get("AO_NVCC_FLAGS", "").encode())
    for f in [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "autooverlap.h")]:
        h.update(f.encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def needs_rebuild():
    """By content, not mtime (a copied tree -- e.g. the snapshot a GPU box runs -- has fresh
    mtimes): the stamp written beside the library must match the current sources."""
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as fh:
        return fh.read().strip() != _source_digest()


def build(force: bool = False, verbose: bool = True) -> str:
    """Compiles every translation unit in parallel (one nvcc per file), then links.  Several
    processes may call this at once (every rank of a torchrun launch does): an exclusive
    file lock serializes them, and a process that waited re-checks before rebuilding."""
    if not force and not needs_rebuild():
        return LIB
    import fcntl
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    with open(os.path.join(ROOT, "build", ".build.lock"), "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        try:
            if not force and not needs_rebuild():
                return LIB
            return _build_locked(verbose)
        finally:
            fcntl.flock(lock, fcntl.LOCK_UN)


def _build_locked(verbose: bool) -> str:
    from concurrent.futures import ThreadPoolExecutor
    digest = _source_digest()  # of the sources this build compiles
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
    tmp = f"{LIB}.{os.getpid()}.tmp"
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    os.replace(tmp, LIB)
    with open(STAMP + ".tmp", "w") as fh:
        fh.write(digest + "\n")
    os.replace(STAMP + ".tmp", STAMP)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
