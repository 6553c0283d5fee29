"""Build libaao.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

Each translation unit is compiled to its own object in parallel (objects are rebuilt only when
their source or a shared header changed), then linked into one shared library.
"""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["csrc/aao.cu", "csrc/kernels_stencil.cu", "csrc/kernels_time.cu", "csrc/kernels_blas.cu",
           "csrc/kernels_freq.cu", "csrc/kernels_kkt.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]
OBJDIR = os.path.join(HERE, "build")


def _headers():
    return [os.path.join(HERE, "csrc", "aao_internal.h"), os.path.join(HERE, "..", "include", "aao.h")]


def _newer(out, deps):
    return os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(d) for d in deps)


def _compile(src, force, verbose):
    obj = os.path.join(OBJDIR, os.path.basename(src).replace(".cu", ".o"))
    if not force and _newer(obj, [src, *_headers()]):
        return obj
    cmd = ["nvcc", *FLAGS, "-c", "-o", obj, src]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=HERE)
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    out = os.path.join(HERE, "libaao.so")
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    if not force and _newer(out, srcs + _headers()):
        return out
    os.makedirs(OBJDIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    cmd = ["nvcc", *ARCH, "-shared", "-o", out, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=HERE)
    return out


if __name__ == "__main__":
    print(build(verbose=True, force=True))
