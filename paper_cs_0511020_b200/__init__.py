"""paper_cs_0511020_b200 -- thin Python binding of libpbit.so (include/pbit.h).

Argument marshalling only: every step of the sort runs in the library's sm_100a
kernels.  PyTorch supplies device memory, streams and process groups.  There is
no CPU fallback: if libpbit.so is missing or fails to load, importing this
package raises.

    head, out_next = sort_list(keys, next, head)                 # device tensors
    head, out_next = sort_list(keys, next, head, out_next=next)  # in place
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PBIT_LIB_PATH") or os.path.join(_HERE, "libpbit.so")  # override: experiments only
PBIT_NULL = 0xFFFFFFFF
NUM_PHASES = 5 + 64
PHASE_NAMES = ["pack", "walk", "rank", "gather", "relink"] + [f"pass{i}" for i in range(64)]
SYMBOLS = ["pbit_sort_list", "pbit_sort_list_mg", "pbit_sort_array", "pbit_mg_get_unique_id", "pbit_mg_comm_init",
           "pbit_mg_comm_destroy", "pbit_mg_comm_abort", "pbit_status_string", "pbit_version", "pbit_last_error",
           "pbit_mg_slice", "pbit_mg_exchange_plan", "pbit_workspace_trim", "pbit_rank_mode", "pbit_mg_transport",
           "pbit_mg_ruler_blocks"]

STATUS = {0: "PBIT_OK", 1: "PBIT_ERR_INVALID_ARG", 2: "PBIT_ERR_INVALID_LIST", 3: "PBIT_ERR_OOM",
          4: "PBIT_ERR_CUDA", 5: "PBIT_ERR_NCCL", 6: "PBIT_ERR_UNSUPPORTED"}


class PbitError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"{STATUS.get(code, code)}{': ' + what if what else ''}")
        self.code = code


class _Opts(ctypes.Structure):
    _fields_ = [("digit_bits", ctypes.c_int), ("stream", ctypes.c_void_p), ("validate", ctypes.c_int),
                ("phase_ms", ctypes.POINTER(ctypes.c_float)), ("passes_run", ctypes.POINTER(ctypes.c_uint32)),
                ("launches", ctypes.POINTER(ctypes.c_uint32)), ("key_kind", ctypes.c_int),
                ("descending", ctypes.c_int), ("out_prev", ctypes.c_void_p), ("out_order", ctypes.c_void_p),
                ("out_keys", ctypes.c_void_p)]


KEY_KINDS = {"unsigned": 0, "signed": 1, "float": 2}  # pbit.h PBIT_KEY_*


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    lib.pbit_sort_list.restype = ctypes.c_int
    lib.pbit_sort_list.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                                   u32p, ctypes.c_void_p, ctypes.POINTER(_Opts)]
    lib.pbit_sort_array.restype = ctypes.c_int
    lib.pbit_sort_array.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.POINTER(_Opts)]
    lib.pbit_sort_list_mg.restype = ctypes.c_int
    lib.pbit_sort_list_mg.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, u32p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.POINTER(_Opts)]
    lib.pbit_mg_get_unique_id.restype = ctypes.c_int
    lib.pbit_mg_get_unique_id.argtypes = [ctypes.c_void_p]
    lib.pbit_mg_comm_init.restype = ctypes.c_int
    lib.pbit_mg_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    lib.pbit_mg_comm_destroy.restype = ctypes.c_int
    lib.pbit_mg_comm_destroy.argtypes = [ctypes.c_void_p]
    lib.pbit_mg_comm_abort.restype = ctypes.c_int
    lib.pbit_mg_comm_abort.argtypes = [ctypes.c_void_p]
    lib.pbit_status_string.restype = ctypes.c_char_p
    lib.pbit_status_string.argtypes = [ctypes.c_int]
    lib.pbit_version.restype = ctypes.c_uint32
    lib.pbit_last_error.restype = ctypes.c_char_p
    lib.pbit_mg_ruler_blocks.restype = ctypes.c_int
    lib.pbit_mg_ruler_blocks.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32),
                                         ctypes.POINTER(ctypes.c_uint32)]
    lib.pbit_mg_transport.restype = ctypes.c_int
    lib.pbit_mg_transport.argtypes = [ctypes.c_void_p]
    lib.pbit_rank_mode.restype = ctypes.c_int
    lib.pbit_rank_mode.argtypes = []
    lib.pbit_workspace_trim.restype = ctypes.c_int
    lib.pbit_workspace_trim.argtypes = [ctypes.c_uint64]
    lib.pbit_mg_slice.restype = ctypes.c_uint64
    lib.pbit_mg_slice.argtypes = [ctypes.c_uint64, ctypes.c_int]
    u64p = ctypes.POINTER(ctypes.c_uint64)
    lib.pbit_mg_exchange_plan.restype = None
    lib.pbit_mg_exchange_plan.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, u64p,
                                          u64p, u64p, u64p, u64p, u64p]
    return lib


lib = _load()

_KEY_BITS = {torch.uint8: 8, torch.int8: 8, torch.int16: 16, torch.uint16: 16, torch.int32: 32,
             torch.uint32: 32, torch.int64: 64, torch.uint64: 64, torch.float16: 16, torch.bfloat16: 16,
             torch.float32: 32, torch.float64: 64}


_FLOAT_DTYPES = (torch.float16, torch.bfloat16, torch.float32, torch.float64)


def _key_kind(keys, key_kind):
    """key_kind=None: "float" for floating-point tensors / arrays, else "unsigned" (integer
    tensors are read as raw unsigned bit patterns: torch's signed dtypes are the usual
    holders of u16/u32/u64 keys -- pass key_kind="signed" for two's complement order).
    An integer order asked for floating-point keys raises instead of sorting raw bits."""
    dt = getattr(keys, "dtype", None)
    is_float = dt in _FLOAT_DTYPES if isinstance(dt, torch.dtype) else getattr(dt, "kind", "") == "f"
    if key_kind is None:
        return "float" if is_float else "unsigned"
    if key_kind not in KEY_KINDS:
        raise ValueError(f"key_kind must be one of {sorted(KEY_KINDS)}")
    if is_float and key_kind != "float":
        raise ValueError(f"key_kind={key_kind!r} for floating-point keys ({dt}): pass key_kind='float' "
                         "or a view of the bits as an integer dtype")
    return key_kind


def rank_mode() -> int:
    """The in-warp ranking the radix passes use on the current device (pbit.h
    pbit_rank_mode): 2 lane-ordered atomics, 0 ballots (self-test fallback)."""
    return int(lib.pbit_rank_mode())


def _errtext(rc: int) -> str:
    t = lib.pbit_status_string(rc).decode()
    if rc in (4, 5):
        t += f" ({lib.pbit_last_error().decode()})"
    return t


def _ptr(t) -> int:
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return t.data_ptr()
    return int(t.ctypes.data)  # numpy (host) array


def _opts(digit_bits: int, stream, phase_ms, passes, launches=None, key_kind: str = "unsigned",
          descending: bool = False):
    o = _Opts()
    o.launches = launches
    o.key_kind = KEY_KINDS[key_kind]
    o.descending = int(bool(descending))
    o.digit_bits = int(digit_bits)
    o.stream = ctypes.c_void_p(stream)
    o.validate = 1
    o.phase_ms = phase_ms
    o.passes_run = passes
    return o


def _stream_handle(stream, on_cuda: bool):
    if stream is not None:
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return torch.cuda.current_stream().cuda_stream if on_cuda and torch.cuda.is_available() else 0


def sort_list(keys, next_, head: int, key_bits: int | None = None, digit_bits: int = 0, out_next=None,
              stream=None, timing: bool = False, key_kind: str | None = None, descending: bool = False,
              out_prev=None, out_order=None, out_keys=None):
    """Stable sort of the list (head, next_) by keys; returns (head, out_next) (plus a
    dict of device ms per phase when timing=True).

    keys / next_ / out_next: CUDA tensors on the current device, or host arrays (torch
    CPU tensors or numpy) -- then the library stages them through device memory.
    next_ holds u32 ids (int32 view, NULL = -1 / 0xFFFFFFFF).  key_kind: "unsigned",
    "signed" or "float" (how the key bits order, pbit.h PBIT_KEY_*; None: inferred, see
    _key_kind); descending: order.
    out_prev (same kind as out_next): also filled with the predecessors of the sorted list
    (doubly-linked lists, pbit.h pbit_opts.out_prev).  out_order / out_keys (same kind as
    out_next): also filled with the node ids / the keys in sorted order (N3 records)."""
    if key_bits is None:
        key_bits = _KEY_BITS[keys.dtype] if isinstance(keys, torch.Tensor) else keys.dtype.itemsize * 8
    key_kind = _key_kind(keys, key_kind)
    n = int(next_.shape[0])
    on_cuda = isinstance(next_, torch.Tensor) and next_.is_cuda
    if out_next is None:
        if isinstance(next_, torch.Tensor):
            out_next = torch.empty_like(next_)
        else:
            import numpy as np
            out_next = np.empty(n, np.uint32)
    oh = ctypes.c_uint32(0)
    pm = (ctypes.c_float * NUM_PHASES)() if timing else None
    passes = ctypes.c_uint32(0)
    launches = ctypes.c_uint32(0)
    o = _opts(digit_bits, _stream_handle(stream, on_cuda), pm, ctypes.pointer(passes), ctypes.pointer(launches),
              key_kind, descending)
    if out_prev is not None and n:
        o.out_prev = ctypes.c_void_p(_ptr(out_prev))
    if out_order is not None and n:
        o.out_order = ctypes.c_void_p(_ptr(out_order))
    if out_keys is not None and n:
        o.out_keys = ctypes.c_void_p(_ptr(out_keys))
    rc = lib.pbit_sort_list(_ptr(keys) if n else None, _ptr(next_) if n else None, head & 0xFFFFFFFF, n, key_bits,
                            ctypes.byref(oh), _ptr(out_next) if n else None, ctypes.byref(o))
    if rc:
        raise PbitError(rc, _errtext(rc))
    if timing:
        ph = {name: float(pm[i]) for i, name in enumerate(PHASE_NAMES) if i < 5 or pm[i] > 0}
        ph["passes_run"] = int(passes.value)
        ph["launches"] = int(launches.value)
        return int(oh.value), out_next, ph
    return int(oh.value), out_next


def sort_array(keys, key_bits: int | None = None, digit_bits: int = 0, out_index=None, out_keys=None,
               want_index: bool = True, want_keys: bool = False, key_kind: str | None = None,
               descending: bool = False, stream=None, timing: bool = False):
    """Stable sort of an ARRAY of keys (pbit.h pbit_sort_array, the paper's "table",
    P:1118-1177).  Returns (out_index, out_keys) -- either may be None -- plus a dict of
    device ms per phase when timing=True.  Tensors on the current CUDA device or host
    arrays (torch CPU tensors or numpy)."""
    if key_bits is None:
        key_bits = _KEY_BITS[keys.dtype] if isinstance(keys, torch.Tensor) else keys.dtype.itemsize * 8
    key_kind = _key_kind(keys, key_kind)
    n = int(keys.shape[0])
    on_cuda = isinstance(keys, torch.Tensor) and keys.is_cuda
    if want_index and out_index is None:
        if isinstance(keys, torch.Tensor):
            out_index = torch.empty(n, dtype=torch.int32, device=keys.device)
        else:
            import numpy as np
            out_index = np.empty(n, np.uint32)
    if want_keys and out_keys is None:
        out_keys = keys.clone() if isinstance(keys, torch.Tensor) else keys.copy()
    pm = (ctypes.c_float * NUM_PHASES)() if timing else None
    passes = ctypes.c_uint32(0)
    launches = ctypes.c_uint32(0)
    o = _opts(digit_bits, _stream_handle(stream, on_cuda), pm, ctypes.pointer(passes), ctypes.pointer(launches),
              key_kind, descending)
    rc = lib.pbit_sort_array(_ptr(keys) if n else None, n, key_bits,
                             _ptr(out_index) if (out_index is not None and n) else None,
                             _ptr(out_keys) if (out_keys is not None and n) else None, ctypes.byref(o))
    if rc:
        raise PbitError(rc, _errtext(rc))
    if timing:
        ph = {name: float(pm[i]) for i, name in enumerate(PHASE_NAMES) if i in (0, 4) or pm[i] > 0}
        ph = {("prep" if k == "pack" else "finish" if k == "relink" else k): v for k, v in ph.items()}
        ph["passes_run"] = int(passes.value)
        ph["launches"] = int(launches.value)
        return out_index, out_keys, ph
    return out_index, out_keys


# ----------------------------------------------------------------------------- multi-GPU
last_mg_launches = 0  # kernels the last sort_list_mg call launched


def workspace_trim(keep_bytes: int = 0) -> None:
    """Release the library's cached workspace on the current device above keep_bytes."""
    rc = lib.pbit_workspace_trim(ctypes.c_uint64(keep_bytes))
    if rc:
        raise PbitError(rc, _errtext(rc))


def mg_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib.pbit_mg_get_unique_id(buf)
    if rc:
        raise PbitError(rc, "ncclGetUniqueId")
    return buf.raw


def mg_comm_init(nranks: int, uid: bytes, rank: int) -> int:
    c = ctypes.c_void_p()
    rc = lib.pbit_mg_comm_init(ctypes.byref(c), nranks, ctypes.c_char_p(uid), rank)
    if rc:
        raise PbitError(rc, "ncclCommInitRank")
    return c.value


def mg_comm_destroy(comm: int) -> None:
    lib.pbit_mg_comm_destroy(ctypes.c_void_p(comm))


def mg_comm_abort(comm: int) -> None:
    """Abort the communicator after sort_list_mg raised PBIT_ERR_NCCL (pbit.h)."""
    lib.pbit_mg_comm_abort(ctypes.c_void_p(comm))


def mg_transport(comm: int) -> str:
    """"peer" (N4: CUDA IPC windows, peer loads and stores), "hybrid" (peer stores, a kn
    replica walked locally) or "nccl": the transport the last sort_list_mg call on `comm`
    used (pbit.h pbit_mg_transport)."""
    return {0: "peer", 1: "nccl", 2: "hybrid"}.get(int(lib.pbit_mg_transport(ctypes.c_void_p(comm))), "none")


def mg_ruler_blocks(n_global: int, nranks: int):
    """(ruler spacing, ruler blocks per rank) of sort_list_mg's walk (pbit.h)."""
    sp, b = ctypes.c_uint32(0), ctypes.c_uint32(0)
    rc = lib.pbit_mg_ruler_blocks(n_global, nranks, ctypes.byref(sp), ctypes.byref(b))
    if rc:
        raise PbitError(rc, "pbit_mg_ruler_blocks")
    return int(sp.value), int(b.value)


def mg_slice(n_global: int, nranks: int) -> int:
    """Node ids per rank for sort_list_mg (ceil(n/G) rounded up to 64)."""
    return int(lib.pbit_mg_slice(n_global, nranks))


def mg_exchange_plan(nranks: int, rank: int, n: int, slice_: int, lt, le):
    """The key-range exchange plan pbit_sort_list_mg computes on the host (see pbit.h):
    returns (send_off, send_count, recv_off, recv_count) for `rank`."""
    import numpy as np
    a = np.ascontiguousarray(lt, dtype=np.uint64).reshape(-1)
    b = np.ascontiguousarray(le, dtype=np.uint64).reshape(-1)
    if a.size == 0:
        a = np.zeros(1, np.uint64)
        b = np.zeros(1, np.uint64)
    outs = [np.zeros(nranks, np.uint64) for _ in range(4)]
    u64p = ctypes.POINTER(ctypes.c_uint64)
    lib.pbit_mg_exchange_plan(nranks, rank, n, slice_, a.ctypes.data_as(u64p), b.ctypes.data_as(u64p),
                              *[o.ctypes.data_as(u64p) for o in outs])
    return tuple(o.astype(np.int64) for o in outs)


def sort_list_mg(keys_local, next_local, head: int, n_global: int, node_lo: int, comm: int,
                 key_bits: int | None = None, digit_bits: int = 0, out_next_local=None, stream=None,
                 key_kind: str | None = None, descending: bool = False, out_prev_local=None,
                 out_order_local=None, out_keys_local=None):
    """Sort one list sharded over the ranks of `comm` (see include/pbit.h).  Returns
    (head, out_next_local)."""
    if key_bits is None:
        key_bits = _KEY_BITS[keys_local.dtype]
    key_kind = _key_kind(keys_local, key_kind)
    n_local = int(next_local.shape[0])
    if out_next_local is None:
        out_next_local = torch.empty_like(next_local)
    oh = ctypes.c_uint32(0)
    launches = ctypes.c_uint32(0)
    o = _opts(digit_bits, _stream_handle(stream, True), None, None, ctypes.pointer(launches), key_kind, descending)
    if out_prev_local is not None and n_local:
        o.out_prev = ctypes.c_void_p(_ptr(out_prev_local))
    if out_order_local is not None and n_local:
        o.out_order = ctypes.c_void_p(_ptr(out_order_local))
    if out_keys_local is not None and n_local:
        o.out_keys = ctypes.c_void_p(_ptr(out_keys_local))
    rc = lib.pbit_sort_list_mg(_ptr(keys_local) if n_local else None, _ptr(next_local) if n_local else None,
                               head & 0xFFFFFFFF, n_global, node_lo, n_local, key_bits, ctypes.byref(oh),
                               _ptr(out_next_local) if n_local else None, ctypes.c_void_p(comm), ctypes.byref(o))
    if rc:
        raise PbitError(rc, _errtext(rc))
    global last_mg_launches
    last_mg_launches = int(launches.value)
    return int(oh.value), out_next_local
