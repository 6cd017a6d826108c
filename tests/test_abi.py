"""The C-ABI library: it loads, exports every symbol include/pbit.h declares, and the
argument checks that need no device behave as the header says.  CPU only."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pbit.h")


@pytest.fixture(scope="module")
def pbit():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_pbit_build", os.path.join(ROOT, "paper_cs_0511020_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()  # rebuilds only when a source is newer than libpbit.so
    import paper_cs_0511020_b200 as p
    return p


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(pbit_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    fns = declared_functions()
    assert "pbit_sort_list" in fns and "pbit_sort_list_mg" in fns


def test_every_declared_symbol_is_exported(pbit):
    lib = ctypes.CDLL(pbit.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(pbit.SYMBOLS)


def test_version_and_status_strings(pbit):
    assert pbit.lib.pbit_version() >= 0x100
    assert pbit.lib.pbit_status_string(2) == b"invalid list"
    assert pbit.lib.pbit_status_string(99) == b"unknown status"


def test_argument_checks_without_device(pbit):
    lib = pbit.lib
    oh = ctypes.c_uint32(7)
    dummy = np.zeros(4, np.uint32)
    p = dummy.ctypes.data
    # out_head NULL
    assert lib.pbit_sort_list(p, p, 0, 4, 32, None, p, None) == 1
    # key width not in {8,16,32,64}
    assert lib.pbit_sort_list(p, p, 0, 4, 24, ctypes.byref(oh), p, None) == 1
    # digit_bits out of range
    for K in (17, -1):
        o = pbit._opts(K, 0, None, None)
        assert lib.pbit_sort_list(p, p, 0, 4, 32, ctypes.byref(oh), p, ctypes.byref(o)) == 1
        assert lib.pbit_sort_array(p, 4, 32, p, None, ctypes.byref(o)) == 1
    # empty list: head must be NULL
    assert lib.pbit_sort_list(None, None, 0xFFFFFFFF, 0, 32, ctypes.byref(oh), None, None) == 0
    assert oh.value == 0xFFFFFFFF
    assert lib.pbit_sort_list(None, None, 0, 0, 32, ctypes.byref(oh), None, None) == 2
    # head >= n, null arrays
    assert lib.pbit_sort_list(p, p, 4, 4, 32, ctypes.byref(oh), p, None) == 1
    assert lib.pbit_sort_list(None, p, 0, 4, 32, ctypes.byref(oh), p, None) == 1
    # n beyond u32 ids
    assert lib.pbit_sort_list(p, p, 0, 1 << 33, 32, ctypes.byref(oh), p, None) == 1


def test_python_wrapper_empty_list(pbit):
    import torch
    h, out = pbit.sort_list(torch.zeros(0, dtype=torch.int32), torch.zeros(0, dtype=torch.int32), 0xFFFFFFFF)
    assert h == 0xFFFFFFFF and out.numel() == 0


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle (DESIGN.md boundary)."""
    pkg = os.path.join(ROOT, "paper_cs_0511020_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(^\s*(import|from)\s+oracle)|(#include\s*[<\"].*oracle)|liboracle|pbit_oracle",
                                     src, flags=re.M), f


def test_key_kind_inferred_from_dtype(pbit):
    """float keys without key_kind sort as floats; an integer order for float
    keys raises instead of sorting raw bit patterns."""
    import torch
    assert pbit._key_kind(torch.zeros(2, dtype=torch.float32), None) == "float"
    assert pbit._key_kind(torch.zeros(2, dtype=torch.bfloat16), None) == "float"
    assert pbit._key_kind(np.zeros(2, np.float64), None) == "float"
    assert pbit._key_kind(torch.zeros(2, dtype=torch.int32), None) == "unsigned"
    assert pbit._key_kind(torch.zeros(2, dtype=torch.int32), "signed") == "signed"
    with pytest.raises(ValueError):
        pbit._key_kind(torch.zeros(2, dtype=torch.float32), "unsigned")
    with pytest.raises(ValueError):
        pbit._key_kind(torch.zeros(2, dtype=torch.int32), "bogus")


def test_header_limits_match_the_checks(pbit):
    """n <= 2^32-2: the header states the limit the library enforces."""
    src = open(HEADER).read()
    assert "2^32-1" not in src
    lib = pbit.lib
    oh = ctypes.c_uint32(7)
    p = np.zeros(4, np.uint32).ctypes.data
    assert lib.pbit_sort_list(p, p, 0, 0xFFFFFFFF, 32, ctypes.byref(oh), p, None) == 1


def test_mg_ruler_blocks_tile_every_slice(pbit):
    """from 2^30 nodes the single-GPU plan spaces rulers 128 apart, but
    a rank's id slice is only a multiple of 64; the multi-GPU walk must use a spacing that
    divides every slice, so that G * blocks * spacing covers all n nodes."""
    for n in [1, 77, 4097, 1 << 24, (1 << 26) + 5, 1 << 30, (1 << 30) + 64, 3_000_000_000, (1 << 32) - 2]:
        for G in [1, 2, 3, 5, 6, 7, 8, 13, 64]:
            S = pbit.mg_slice(n, G)
            if G * S > 0xFFFFFFFF:
                with pytest.raises(pbit.PbitError):
                    pbit.mg_ruler_blocks(n, G)
                continue
            sp, b = pbit.mg_ruler_blocks(n, G)
            assert sp & (sp - 1) == 0 and sp <= 64 and S % sp == 0
            assert b == S // sp and G * b * sp >= n


def test_header_is_plain_c_and_the_example_links(pbit, tmp_path):
    """include/pbit.h compiles as C99 and a plain C program links against libpbit.so
    (examples/sort_list.c; it runs on a GPU box: tests/test_gpu_parity.py)."""
    import subprocess
    exe = tmp_path / "sort_list"
    libdir = os.path.dirname(os.path.abspath(pbit.LIB_PATH))
    r = subprocess.run(["cc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "sort_list.c"), os.path.abspath(pbit.LIB_PATH),
                        f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
