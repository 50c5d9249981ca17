"""Build libchkpcg.so in-tree with nvcc for sm_100a (no JIT cache, no pip install)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libchkpcg.so")
SOURCES = [os.path.join(SRC, "chk_capi.cu")]
DEPS = SOURCES + [os.path.join(SRC, f) for f in ("chk_fft.cuh", "chk_kernels.cuh", "chk_tma.cuh", "chk_plane.cuh", "chk_sample.cuh")] + [
    os.path.join(REPO, "include", "chk_pcg.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-diag-suppress", "177",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", os.path.join(REPO, "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and up_to_date():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT, *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
