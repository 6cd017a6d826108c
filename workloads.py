"""workloads.py -- seeded synthetic linked lists shaped like the paper's workloads.

This module is the ONLY code shared by the oracle side (tests, oracle/) and the
CUDA side (bench.py, GPU tests).  It holds none of the method's arithmetic: no
digit extraction, no counting, no ordering.  It only draws keys and link orders.

All draws are counter-based integer hashes computed with torch int64 ops that
never overflow (every product is < 2^63), so the same (config, seed) gives
bit-identical arrays on CPU and on CUDA.

Representation handed to both sides:
  keys  : node-indexed, torch dtype uint8 / int16 / int32 / int64 holding the
          unsigned 8/16/32/64-bit key bit pattern
  next  : node-indexed int32 holding the u32 successor id, NULL = -1 (0xFFFFFFFF)
  head  : python int (0xFFFFFFFF for the empty list)
  order : int64 list order, order[p] = node at list position p (so the input
          rank of node v is the p with order[p] == v; used only by checkers)

Paper workload context: keys from C rand() with RAND_MAX = 0x7FFF and lists built
by push.  The BASELINE.json configs C1..C5 are the headline
shapes; the paper-shaped "ctx" config reproduces P:836-842.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

NULL32 = 0xFFFFFFFF
_M32 = 0xFFFFFFFF


# --------------------------------------------------------------------------- hashing
def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for 0 <= x < 2^32 without int64 overflow."""
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & _M32


def hash32(x: torch.Tensor, seed: int) -> torch.Tensor:
    """A keyed 32-bit avalanche hash (xorshift-multiply, 'lowbias32' constants)."""
    x = (x ^ (seed & _M32)) & _M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    x = _mul32(x, 0x9E3779B1 ^ ((seed >> 32) & 0xFFFF))
    x = x ^ (x >> 16)
    return x


def _stream(i: torch.Tensor, seed: int, stream: int) -> torch.Tensor:
    return hash32(hash32(i & _M32, seed * 0x9E37 + stream) ^ ((i >> 32) & _M32), seed + 0x5bd1e995 * stream)


def _bijection_bits(x: torch.Tensor, bits: int, seed: int) -> torch.Tensor:
    """A keyed bijection on [0, 2^bits): rounds of odd-multiply, xor-shift, add."""
    mask = (1 << bits) - 1
    if bits == 0:
        return x
    for r in range(6):
        k = int(hash32(torch.tensor([r], dtype=torch.int64), seed)[0])
        odd = (k | 1) & mask
        x = _mul32(x, odd) & mask
        x = x ^ (x >> max(1, (bits + 1) // 2))
        x = (x + (k >> 3)) & mask
        x = x ^ (x >> max(1, bits // 3))
    return x


CHUNK = 1 << 24  # elements per generator chunk: every draw is per element (or per 4096-run), so
#                 chunking bounds the temporaries without changing a single value


def _perm_values(x: torch.Tensor, n: int, bits: int, seed: int) -> torch.Tensor:
    y = _bijection_bits(x, bits, seed)
    bad = y >= n
    while bool(bad.any()):
        y[bad] = _bijection_bits(y[bad], bits, seed)
        bad = y >= n
    return y


def _perm_bits(n: int) -> int:
    return max(1, math.ceil(math.log2(n))) if n > 1 else 1


def permutation_range(a: int, b: int, n: int, seed: int, device="cpu") -> torch.Tensor:
    """Entries [a, b) of permutation(n, seed) (int64), computed on their own."""
    return _perm_values(torch.arange(a, b, dtype=torch.int64, device=device), n, _perm_bits(n), seed)


def permutation(n: int, seed: int, device="cpu") -> torch.Tensor:
    """A seeded pseudo-random permutation of [0, n) (int64), by cycle-walking a keyed
    bijection on the enclosing power of two.  Same result on every device."""
    out = torch.empty(n, dtype=torch.int64, device=device)
    for a in range(0, n, CHUNK):
        b = min(n, a + CHUNK)
        out[a:b] = permutation_range(a, b, n, seed, device)
    return out


def uniform_u32(n: int, seed: int, stream: int, device="cpu") -> torch.Tensor:
    return _stream(torch.arange(n, dtype=torch.int64, device=device), seed, stream)


# --------------------------------------------------------------------------- lists
@dataclass
class ListInput:
    keys: torch.Tensor
    next: torch.Tensor
    head: int
    order: torch.Tensor
    key_bits: int
    payload: torch.Tensor | None = None
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.next.shape[0])


_KEY_TORCH = {8: torch.uint8, 16: torch.int16, 32: torch.int32, 64: torch.int64}


def to_key_tensor(k_int64: torch.Tensor, key_bits: int, hi: torch.Tensor | None = None) -> torch.Tensor:
    """Pack unsigned values held in int64 (and an optional high 32-bit word for
    64-bit keys) into the torch storage dtype for key_bits."""
    if key_bits == 8:
        return k_int64.to(torch.uint8)
    if key_bits == 16:
        return (k_int64 - ((k_int64 >= 1 << 15).to(torch.int64) << 16)).to(torch.int16)
    if key_bits == 32:
        return (k_int64 - ((k_int64 >= 1 << 31).to(torch.int64) << 32)).to(torch.int32)
    assert hi is not None
    # (hi << 32) | lo as a two's-complement int64: hi in [0,2^32) -> signed high word
    hs = hi - ((hi >= 1 << 31).to(torch.int64) << 32)
    return (hs << 32) | k_int64


def links_from_order(order: torch.Tensor, n: int) -> tuple[torch.Tensor, int]:
    """next[order[p]] = order[p+1], next[order[n-1]] = NULL, head = order[0]."""
    nxt = torch.full((n,), -1, dtype=torch.int32, device=order.device)
    if n == 0:
        return nxt, NULL32
    nxt[order[:-1]] = order[1:].to(torch.int32)
    return nxt, int(order[0])


def link_order(n: int, kind: str, seed: int, device="cpu") -> torch.Tensor:
    """List order (position -> node id).
    random   : a seeded random permutation (BASELINE.json C1-C5)
    identity : next[v] = v+1 (head 0)
    push     : next[v] = v-1, head n-1 -- a list built by push
    """
    if kind == "random":
        return permutation(n, seed, device)
    if kind == "identity":
        return torch.arange(n, dtype=torch.int64, device=device)
    if kind == "push":
        return torch.arange(n - 1, -1, -1, dtype=torch.int64, device=device)
    raise ValueError(kind)


def zipf_thresholds(num_values: int, s: float) -> np.ndarray:
    """Inverse-CDF table for Zipf(s) over ranks 1..num_values as integer thresholds in
    [0, 2^32] (float64 CDF built on the host, so every device draws identically)."""
    r = np.arange(1, num_values + 1, dtype=np.float64)
    w = r ** (-s)
    cdf = np.cumsum(w) / w.sum()
    thr = np.floor(cdf * 4294967296.0).astype(np.int64)
    thr[-1] = 1 << 32
    return thr


_I64_MIN = -(1 << 63)


def _ordered(lo: torch.Tensor, hi: torch.Tensor | None, key_bits: int) -> torch.Tensor:
    """int64 whose signed order is the unsigned order of the key (lo, hi): the key itself
    below 64 bits, the 64-bit pattern with its top bit flipped otherwise."""
    return lo if key_bits < 64 else to_key_tensor(lo, 64, hi) ^ _I64_MIN


def _from_ordered(c: torch.Tensor, key_bits: int) -> torch.Tensor:
    return to_key_tensor(c, key_bits) if key_bits < 64 else c ^ _I64_MIN


def _key_chunk(a: int, b: int, key_bits: int, seed: int, keys: str, key_range, thr, device) -> torch.Tensor:
    """Keys of list positions [a, b), as the int64 `_ordered` form.  Per position, except
    'runs4096' (per run of 4096 positions; a must be a multiple of 4096)."""
    pos = torch.arange(a, b, dtype=torch.int64, device=device)
    lo = _stream(pos, seed, 1)
    hi = _stream(pos, seed, 2) if key_bits == 64 else None
    mask = (1 << min(key_bits, 32)) - 1
    if keys == "uniform":
        if key_range is not None:
            assert key_range <= 1 << 32
            lo = lo % key_range if key_range & (key_range - 1) else lo & (key_range - 1)
            if hi is not None:
                hi = torch.zeros_like(hi)
        else:
            lo = lo & mask
    elif keys == "zipf":
        rank = torch.searchsorted(thr, lo, right=True)  # 0-based rank
        lo = _bijection_bits(rank, 32, seed ^ 0x2222) & mask
        if hi is not None:
            hi = torch.zeros_like(hi)
    elif keys == "equal":
        lo = torch.full_like(lo, 0x5A5A5A5A & mask)
        if hi is not None:
            hi = torch.full_like(hi, 0x5A5A5A5A)
    elif keys == "max":
        lo = torch.full_like(lo, mask)
        if hi is not None:
            hi = torch.full_like(hi, _M32)
    elif keys in ("sorted", "reverse", "runs4096"):
        lo = lo & mask
    else:
        raise ValueError(keys)
    comb = _ordered(lo, hi, key_bits)
    if keys == "runs4096":
        # alternating presorted / random runs of 4096 list positions (reading Q12): runs
        # with an even global index are sorted ascending (by the full unsigned key)
        run = 4096
        assert a % run == 0
        full = ((b - a) // run) * run
        if full:
            blocks = comb[:full].view(-1, run)
            srt = torch.sort(blocks, dim=1).values
            first = a // run
            is_p = ((torch.arange(blocks.shape[0], device=device) + first) % 2 == 0).unsqueeze(1)
            comb[:full] = torch.where(is_p, srt, blocks).reshape(-1)
    return comb


def make_list(n: int, key_bits: int, seed: int, keys: str = "uniform", links: str = "random",
              device="cpu", key_range: int | None = None, zipf_s: float = 1.1,
              zipf_values: int = 1 << 20) -> ListInput:
    """General seeded list generator used by tests and bench.

    keys: 'uniform' (full key_bits range, or [0, key_range)), 'zipf' (Zipf(zipf_s) rank
    over zipf_values values, mapped to a 32-bit value by a keyed bijection -- DESIGN.md
    reading Q17), 'equal' (all keys 0x5A..), 'max' (all ones), 'sorted'/'reverse'
    (along the list), 'runs4096' (C4: alternating presorted / random runs of 4096 list
    positions, reading Q12).  64-bit keys use all 64 bits in every kind that draws them.

    Everything is drawn per list position (or per run of 4096 positions) in chunks of
    CHUNK positions, so large lists need no full-size temporaries; the values do not
    depend on the chunking or on the device.
    """
    order = link_order(n, links, seed ^ 0x1111, device)
    thr = torch.from_numpy(zipf_thresholds(zipf_values, zipf_s)).to(device) if keys == "zipf" else None
    key = torch.empty(n, dtype=_KEY_TORCH[key_bits], device=device)   # node-indexed
    if keys in ("sorted", "reverse"):  # a global sort along the list (small lists only)
        comb = _key_chunk(0, n, key_bits, seed, keys, None, None, device)
        comb = torch.sort(comb, descending=(keys == "reverse")).values
        key[order] = _from_ordered(comb, key_bits)
    else:
        for a in range(0, n, CHUNK):
            b = min(n, a + CHUNK)
            key[order[a:b]] = _from_ordered(_key_chunk(a, b, key_bits, seed, keys, key_range, thr, device),
                                            key_bits)
    nxt, head = links_from_order(order, n)
    payload = None
    if keys == "runs4096" or key_bits == 64:
        payload = torch.empty(n, dtype=torch.int64, device=device)
        for a in range(0, n, CHUNK):
            v = torch.arange(a, min(n, a + CHUNK), dtype=torch.int64, device=device)
            payload[a:a + v.shape[0]] = to_key_tensor(_stream(v, seed, 7), 64, _stream(v, seed, 8))
    return ListInput(keys=key, next=nxt, head=head, order=order, key_bits=key_bits,
                     payload=payload, name=f"n={n},u{key_bits},{keys},{links}")


# --------------------------------------------------------------------------- configs
# BASELINE.json configs (C1..C5) and the paper-shaped context workload.  Seeds fixed.
CONFIGS = {
    "C1": dict(n=1 << 16, key_bits=8, keys="uniform", links="random", digit_bits=4, seed=101,
               desc="n=65536, u8 uniform [0,255], random-permutation links, K=4"),
    "C2": dict(n=1 << 24, key_bits=32, keys="uniform", links="random", digit_bits=8, seed=202,
               desc="n=2^24, u32 uniform, random-permutation links"),
    "C3": dict(n=1 << 28, key_bits=32, keys="zipf", links="random", digit_bits=8, seed=303,
               desc="n=2^28, u32 Zipf(1.1) over 2^20 values, random-permutation links"),
    "C4": dict(n=1 << 27, key_bits=64, keys="runs4096", links="random", digit_bits=8, seed=404,
               desc="n=2^27, u64 uniform + u64 payload, 50% presorted runs of 4096"),
    "C5": dict(n=1 << 30, key_bits=32, keys="uniform", links="random", digit_bits=8, seed=505,
               key_range=1 << 16, desc="n=2^30, u32 uniform in [0,2^16), random-permutation links"),
    "ctx": dict(n=10_000_000, key_bits=32, keys="uniform", links="push", digit_bits=4, seed=606,
                key_range=0x8000, desc="paper-shaped: n=1e7, rand() keys in [0,0x7FFF], push-built list"),
}


def make_config(name: str, device="cpu", n: int | None = None, seed: int | None = None) -> ListInput:
    c = dict(CONFIGS[name])
    li = make_list(n if n is not None else c["n"], c["key_bits"], c["seed"] if seed is None else seed,
                   keys=c["keys"], links=c["links"], device=device, key_range=c.get("key_range"))
    li.name = name
    return li


# --------------------------------------------------------------------------- numpy views
def keys_numpy(li: ListInput) -> np.ndarray:
    k = li.keys.cpu().numpy()
    return k.view({8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[li.key_bits])


def next_numpy(li: ListInput) -> np.ndarray:
    return li.next.cpu().numpy().view(np.uint32)
