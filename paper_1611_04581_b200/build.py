"""Builds the in-tree C-ABI library libdsgd_b200.so for sm_100a with nvcc.

    python -m paper_1611_04581_b200.build      (or __graft_entry__.build())

The .so lands next to this file so it travels with the repo snapshot to the
GPU box (it is git-ignored, not gpurun-ignored).  The translation units are
compiled in parallel (the kernels once per dtype) and linked with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libdsgd_b200.so")
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in
           ("dsgd_kernels.cu", "dsgd_runtime.cu", "dsgd_rng.cpp", "dsgd_multicast.cpp")]
HEADERS = [os.path.join(CSRC, f) for f in
           ("dsgd_device.cuh", "dsgd_kernels.cuh", "dsgd_internal.h")] + \
          [os.path.join(ROOT, "include", "dsgd_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# (source, extra defines) -> one object each
UNITS = [("dsgd_kernels.cu", ["-DDSGD_KERNEL_DTYPE=32"]),
         ("dsgd_kernels.cu", ["-DDSGD_KERNEL_DTYPE=64"]),
         ("dsgd_runtime.cu", []),
         ("dsgd_rng.cpp", []),
         ("dsgd_multicast.cpp", [])]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS if os.path.exists(f))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    common = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    if verbose:
        common.insert(0, "-Xptxas=-v")
    with tempfile.TemporaryDirectory(prefix="dsgd_build_") as tmp:
        procs, objs = [], []
        for i, (src, defs) in enumerate(UNITS):
            path = os.path.join(CSRC, src)
            if not os.path.exists(path):
                continue
            obj = os.path.join(tmp, f"u{i}.o")
            cmd = [NVCC, *common, *defs, "-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd))
            procs.append((cmd, subprocess.Popen(cmd)))
            objs.append(obj)
        failed = [cmd for cmd, p in procs if p.wait() != 0]
        if failed:
            raise subprocess.CalledProcessError(1, failed[0])
        # host linker: no device-link step (no relocatable device code), so
        # each object's cubin is embedded once
        cuda = os.path.dirname(os.path.dirname(os.path.realpath(NVCC)))
        link = ["g++", "-shared", *objs, "-o", SO + ".tmp", "-L" + os.path.join(cuda, "lib64"),
                "-lcudart_static", "-lnccl", "-ldl", "-lrt", "-lpthread"]
        subprocess.run(link, check=True)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
