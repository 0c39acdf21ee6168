"""Builds the in-tree C-ABI library libdsgd_b200.so for sm_100a with nvcc.

    python -m paper_1611_04581_b200.build      (or __graft_entry__.build())

The .so lands next to this file so it travels with the repo snapshot to the
GPU box (it is git-ignored, not gpurun-ignored)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libdsgd_b200.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in
           ("dsgd_kernels.cu", "dsgd_runtime.cu", "dsgd_rng.cpp")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in
           ("dsgd_device.cuh", "dsgd_kernels.cuh", "dsgd_internal.h")] + \
          [os.path.join(ROOT, "include", "dsgd_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "csrc"),
           *SOURCES, "-o", SO + ".tmp", "-lnccl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
