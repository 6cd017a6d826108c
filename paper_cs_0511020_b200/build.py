"""Build libpbit.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpbit.so")
SOURCES = ["pbit.cu", "mg.cu"]
HEADERS = ["common.cuh", "kernels.cuh", "pbit_internal.h", "launch.cuh", "mg_kernels.cuh", "small.cuh"]


def nccl_dirs():
    import nvidia.nccl  # torch's NCCL (2.28.x): link the one torch loads
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc_cmd(out=LIB, extra=()):
    inc, lib = nccl_dirs()
    return ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC,-O2", "-shared", "-Xptxas", "-v" if os.environ.get("PBIT_PTXAS_V") else "-O3",
            f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}",
            *[os.path.join(CSRC, s) for s in SOURCES],
            f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={lib}", *extra, "-o", out]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "pbit.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = nvcc_cmd(tmp)
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="-f" in sys.argv, verbose=True)
