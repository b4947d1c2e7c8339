"""In-tree build of the CUDA engine (``lib/libcace_gpu.so``) for sm_100a.

``python -m paper_2506_18796_b200.build`` (or ``__graft_entry__.build()``).
nvcc cross-compiles here without a GPU; the .so travels with the repo
snapshot to the GPU box.

Flags: ``-fmad=false`` (the reference is built without FMA contraction, so
every fp64 op must round separately — the glibc-log restatement issues its
own explicit __fma_rn), ``-Xcompiler -ffp-contract=off`` for the host-side
restatement, ``-lineinfo`` so ncu's source page maps to the kernels.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libcace_gpu.so")
SOURCES = [os.path.join(CSRC, "capi.cu")]
DEPS = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
    os.path.join(HERE, "..", "include", "cace_gpu.h")]

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-fmad=false", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT + ".tmp", *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
