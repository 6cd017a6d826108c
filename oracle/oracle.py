"""ctypes binding of oracle/pbit_oracle.c -- TEST INFRASTRUCTURE ONLY.

Marshals numpy arrays into the C oracle; holds none of the method's arithmetic.
The shared object is compiled with gcc on first use (or by
``__graft_entry__.build()``); building the checker is not using it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

ORACLE_NULL = 0xFFFFFFFF
_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pbit_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__({1: "invalid argument", 2: "invalid list", 3: "out of memory"}.get(code, str(code)))
        self.code = code


class Counters(ctypes.Structure):
    _fields_ = [
        ("relinks", ctypes.c_uint64),
        ("merge_visits", ctypes.c_uint64),
        ("max_depth", ctypes.c_uint32),
        ("max_live_tabs", ctypes.c_uint32),
        ("bucket_scans", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, plain C11) if missing or stale."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            u32p = ctypes.POINTER(ctypes.c_uint32)
            lib.oracle_pbit_sort.restype = ctypes.c_int
            lib.oracle_pbit_sort.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32,
                                             ctypes.c_uint64, ctypes.c_uint, ctypes.c_int, u32p,
                                             ctypes.c_void_p, ctypes.POINTER(Counters)]
            lib.oracle_pbit_sort_kind.restype = ctypes.c_int
            lib.oracle_pbit_sort_kind.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32,
                                                  ctypes.c_uint64, ctypes.c_uint, ctypes.c_int, ctypes.c_int, u32p,
                                                  ctypes.c_void_p, ctypes.POINTER(Counters)]
            lib.oracle_repair_back.restype = ctypes.c_int
            lib.oracle_repair_back.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p]
            lib.oracle_split_once.restype = ctypes.c_int
            lib.oracle_split_once.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32,
                                              ctypes.c_uint64, ctypes.c_uint, ctypes.c_void_p]
            lib.oracle_validate_list.restype = ctypes.c_int
            lib.oracle_validate_list.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64]
            lib.oracle_pbit_sort_par.restype = ctypes.c_int
            lib.oracle_pbit_sort_par.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32,
                                                 ctypes.c_uint64, ctypes.c_uint, ctypes.c_int, u32p, ctypes.c_void_p]
            lib.oracle_list_order.restype = ctypes.c_int
            lib.oracle_list_order.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p]
            lib.oracle_bits.restype = ctypes.c_uint64
            lib.oracle_bits.argtypes = [ctypes.c_uint64, ctypes.c_uint, ctypes.c_uint]
            lib.oracle_memory_bound_T.restype = ctypes.c_uint64
            lib.oracle_memory_bound_T.argtypes = [ctypes.c_uint, ctypes.c_uint]
            _lib = lib
    return _lib


_KEY_DTYPES = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}


def _keys(keys, key_bits):
    k = np.ascontiguousarray(keys)
    want = _KEY_DTYPES.get(key_bits)
    if want is None:  # let the C side reject the width (ORACLE_ERR_ARG)
        return k
    if k.dtype != want:
        # same-width signed / float keys: pass the bit patterns unchanged
        k = k.view(want) if k.dtype.itemsize * 8 == key_bits else k.astype(want)
    return k


KINDS = {"unsigned": 0, "signed": 1, "float": 2}


def pbit_sort(keys, next_, head: int, key_bits: int, K: int = 4, descending: bool = False,
              with_counters: bool = False, out=None, kind: str = "unsigned"):
    """Return (out_head, out_next[, counters]) of the paper-literal Pbit sort.
    ``out`` (uint32, contiguous) may be ``next_`` itself: the sort relinks in situ.
    ``kind``: "unsigned", "signed" (the dispatcher P:444-466, reading Q13) or
    "float" (IEEE 754 binary16/32/64 by key_bits: mantissa then characteristic, P:1190,
    reading Q18).  Keys are passed as their bit patterns (any dtype of key_bits width)."""
    lib = _load()
    nxt = np.ascontiguousarray(next_, dtype=np.uint32)
    n = int(nxt.shape[0])
    k = _keys(keys, key_bits) if n else np.zeros(1, _KEY_DTYPES.get(key_bits, np.uint8))
    if out is None:
        out = np.empty(max(n, 1), np.uint32)
    else:
        assert out.dtype == np.uint32 and out.flags.c_contiguous and out.shape[0] >= n
    oh = ctypes.c_uint32(0)
    c = Counters()
    rc = lib.oracle_pbit_sort_kind(k.ctypes.data, key_bits, nxt.ctypes.data if n else None, head & 0xFFFFFFFF,
                                   n, K, KINDS[kind], int(descending), ctypes.byref(oh), out.ctypes.data,
                                   ctypes.byref(c))
    if rc:
        raise OracleError(rc)
    res = (int(oh.value), out[:n])
    return res + (c.as_dict(),) if with_counters else res


def pbit_sort_par(keys, next_, head: int, key_bits: int, K: int = 4, threads: int = 0):
    """The same ascending sort with the recursion below the first two levels on `threads`
    host threads (0 = every core); bit-identical to pbit_sort.  Returns (out_head, out_next)."""
    lib = _load()
    nxt = np.ascontiguousarray(next_, dtype=np.uint32)
    n = int(nxt.shape[0])
    k = _keys(keys, key_bits) if n else np.zeros(1, _KEY_DTYPES.get(key_bits, np.uint8))
    out = np.empty(max(n, 1), np.uint32)
    oh = ctypes.c_uint32(0)
    rc = lib.oracle_pbit_sort_par(k.ctypes.data, key_bits, nxt.ctypes.data if n else None, head & 0xFFFFFFFF, n, K,
                                  threads, ctypes.byref(oh), out.ctypes.data)
    if rc:
        raise OracleError(rc)
    return int(oh.value), out[:n]


def repair_back(next_, head: int):
    """The doubly-linked "reverse connection" repair after sorting:
    returns back[] with back[v] = the node right behind v (NULL for the head)."""
    nxt = np.ascontiguousarray(next_, dtype=np.uint32)
    back = np.empty(max(nxt.shape[0], 1), np.uint32)
    rc = _load().oracle_repair_back(nxt.ctypes.data if nxt.size else None, head & 0xFFFFFFFF, nxt.shape[0],
                                    back.ctypes.data)
    if rc:
        raise OracleError(rc)
    return back[:nxt.shape[0]]


def split_once(keys, next_, head: int, key_bits: int, K: int = 4):
    """First split of P:351-353: returns (tab heads, relinked next)."""
    lib = _load()
    nxt = np.array(next_, dtype=np.uint32, copy=True)
    k = _keys(keys, key_bits)
    tab = np.empty(1 << K, np.uint32)
    rc = lib.oracle_split_once(k.ctypes.data, key_bits, nxt.ctypes.data, head & 0xFFFFFFFF,
                               nxt.shape[0], K, tab.ctypes.data)
    if rc:
        raise OracleError(rc)
    return tab, nxt


def validate_list(next_, head: int) -> bool:
    nxt = np.ascontiguousarray(next_, dtype=np.uint32)
    return _load().oracle_validate_list(nxt.ctypes.data if nxt.size else None, head & 0xFFFFFFFF,
                                        nxt.shape[0]) == 0


def list_order(next_, head: int):
    """order[i] = the i-th node of the list (head, next_): the traversal L = L->next."""
    nxt = np.ascontiguousarray(next_, dtype=np.uint32)
    order = np.empty(max(nxt.shape[0], 1), np.uint32)
    rc = _load().oracle_list_order(nxt.ctypes.data if nxt.size else None, head & 0xFFFFFFFF, nxt.shape[0],
                                   order.ctypes.data)
    if rc:
        raise OracleError(rc)
    return order[:nxt.shape[0]]


def bits(number: int, M: int, K: int = 4) -> int:
    return int(_load().oracle_bits(number, M, K))


def memory_bound_T(M: int, K: int) -> int:
    return int(_load().oracle_memory_bound_T(M, K))
