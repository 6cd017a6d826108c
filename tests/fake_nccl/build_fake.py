"""TEST INFRASTRUCTURE: build libpbit_fakenccl.so -- the product sources (pbit.cu, mg.cu)
linked with fake_nccl.cpp instead of NCCL, so G ranks can run pbit_sort_list_mg's real
kernels and host code as G threads on one GPU (tests/fake_nccl/run_mg_threads.py)."""
from __future__ import annotations

import importlib.util
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "libpbit_fakenccl.so")
FAKE = os.path.join(HERE, "fake_nccl.cpp")


def _product_build():
    spec = importlib.util.spec_from_file_location("_pbit_build", os.path.join(ROOT, "paper_cs_0511020_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b


def build(force: bool = False) -> str:
    """PBIT_BOUNDS_CHECK=1 in the environment: the objects with device-side bounds checks
    (their own objdir and library)."""
    b = _product_build()
    bounds = os.environ.get("PBIT_BOUNDS_CHECK") == "1"
    out = OUT.replace(".so", "_bounds.so") if bounds else OUT
    objs = (b.objects(extra=["-DPBIT_BOUNDS_CHECK=1"], objdir=b.OBJDIR + "_bounds") if bounds
            else b.objects())  # the product's own objects (compiled once, shared with libpbit.so)
    if not force and not b._newer(out, objs + [FAKE, __file__]):
        return out
    inc, _ = b.nccl_dirs()
    fobj = os.path.join(b.OBJDIR, "fake_nccl.o")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", f"-I{inc}", "-I/usr/local/cuda/include",
                           "-c", FAKE, "-o", fobj])
    b.link(out, objs + [fobj], link_nccl=False, extra=["-Xlinker", "-Bsymbolic"])
    return out


if __name__ == "__main__":
    print(build(force="-f" in sys.argv))
