"""Build libaao.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["csrc/aao.cu", "csrc/kernels_stencil.cu", "csrc/kernels_time.cu", "csrc/kernels_blas.cu",
           "csrc/kernels_freq.cu"]
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills"]


def build(verbose: bool = False, force: bool = False) -> str:
    out = os.path.join(HERE, "libaao.so")
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    deps = srcs + [os.path.join(HERE, "csrc", "aao_internal.h"), os.path.join(HERE, "..", "include", "aao.h")]
    if not force and os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(d) for d in deps):
        return out
    cmd = ["nvcc", *FLAGS, "-o", out, *srcs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=HERE)
    return out


if __name__ == "__main__":
    print(build(verbose=True, force=True))
