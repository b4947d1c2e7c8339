"""In-tree build of the CUDA engine (``lib/libcace_gpu.so``) for sm_100a.

``python paper_2506_18796_b200/build.py`` (or ``__graft_entry__.build()``); running it
as a script does not import the package, which refuses to load without the
library.
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


def build(force: bool = False, verbose: bool = False, out: str = OUT) -> str:
    if out != OUT:
        return _build_to(out, verbose)
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    extra = os.environ.get("CACE_NVCC_EXTRA", "").split()  # experiments, e.g. -DCACE_LANE_MIN_BLOCKS=5
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", OUT + ".tmp", *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


def _build_to(out: str, verbose: bool) -> str:
    extra = os.environ.get("CACE_NVCC_EXTRA", "").split()
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", out, *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    print(build(force="--force" in sys.argv, verbose=True, out=os.path.abspath(args[0]) if args else OUT))
