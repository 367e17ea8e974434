"""Build libising.so (sm_100a) in-tree with nvcc.  Called by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libising.so")
SOURCES = ["ising_kernels.cu", "ising_basic.cu", "ising_runtime.cu"]
HEADERS = ["ising_kernels.cuh", os.path.join("..", "..", "include", "ising.h")]


def nccl_dir() -> str:
    for base in [sysconfig.get_paths()["purelib"], *sys.path]:
        d = os.path.join(base, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers (nvidia/nccl) not found in site-packages")


def nvcc() -> str:
    for c in [os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"]:
        if c and os.path.exists(c):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nd = nccl_dir()
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [
        nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
        "-I", os.path.join(nd, "include"), "-I", os.path.join(ROOT, "include"),
        *[os.path.join(CSRC, f) for f in SOURCES],
        "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-ldl",
        "-Xlinker", "-rpath=" + os.path.join(nd, "lib"),
        "-o", tmp,
    ]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
