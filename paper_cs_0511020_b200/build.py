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


def nvcc_cmd(out=LIB, extra=(), link_nccl=True):
    """link_nccl=False: NCCL headers only (the test build that links a stand-in)."""
    inc, lib = nccl_dirs()
    link = [f"-L{lib}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"] if link_nccl else []
    return ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC,-O2", "-shared", "-Xptxas", "-v" if os.environ.get("PBIT_PTXAS_V") else "-O3",
            f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}",
            *[os.path.join(CSRC, s) for s in SOURCES],
            *link, *extra, "-o", out]


OBJDIR = os.path.join(ROOT, "build", "obj")


def _common_flags():
    inc, _ = nccl_dirs()
    return ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v" if os.environ.get("PBIT_PTXAS_V") else "-O3",
            f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}"]


def _deps():
    return [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "pbit.h"), __file__]


def _newer(target, deps):
    return not os.path.exists(target) or any(os.path.getmtime(d) > os.path.getmtime(target) for d in deps)


def objects(force: bool = False, verbose: bool = False, extra=(), objdir: str = OBJDIR) -> list:
    """Compile each source to build/obj/<name>.o, in parallel (the two sources take about
    the same time); shared by libpbit.so and the tests' fake-NCCL build.  `extra` flags
    (e.g. -DPBIT_BOUNDS_CHECK=1) go with their own objdir."""
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        if force or _newer(obj, _deps()):
            cmd = ["nvcc", *_common_flags(), *extra, "-c", os.path.join(CSRC, src), "-o", obj + f".tmp{os.getpid()}"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append((obj, subprocess.Popen(cmd)))
    bad = [o for o, p in procs if p.wait() != 0]
    if bad:
        raise RuntimeError(f"nvcc failed: {bad}")
    for o, _ in procs:
        os.replace(o + f".tmp{os.getpid()}", o)
    return objs


def link(out: str, objs: list, link_nccl: bool = True, extra=()) -> None:
    _, lib = nccl_dirs()
    nccl = [f"-L{lib}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"] if link_nccl else []
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, *nccl,
                           *extra, "-o", tmp])
    os.replace(tmp, out)


def stale():
    return _newer(LIB, _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        objs = objects(force=force, verbose=verbose)
        link(LIB, objs)
    return LIB


if __name__ == "__main__":
    build(force="-f" in sys.argv, verbose=True)
