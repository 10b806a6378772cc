"""Seeded synthetic inputs shared by the parity tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic: it only turns
(seed, stream key, element index) into numbers.  It is the one module both the
oracle side and the CUDA side draw inputs from.

Generator: SplitMix64 in counter mode.  Element e of stream `key` is
    out(e) = mix64(skey + (e + 1) * GAMMA),  skey = mix64(seed ^ mix64(key)),
evaluated identically by the pure-numpy path (host) and by torch int64 ops on
any device (wrapping 64-bit arithmetic, logical shifts emulated by masking).
The stream is keyed by the GLOBAL element index, so a shard [lo, hi) of a batch
is bit-identical to the same slice of the unsharded batch.

Distributions:
  * "uniform": U[-1, 1) per real component; fp64 uses 53 random bits
    (multiples of 2^-52), fp32 uses 24 random bits (multiples of 2^-23) -- both
    exactly representable, so the same stream gives the same values on every
    device.
  * "int": integers in [-4, 4] (exact-arithmetic parity cases).
"""
from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1
DEFAULT_SEED = 13047053

_KIND_DT = {"s": ("f32", False), "d": ("f64", False), "c": ("f32", True), "z": ("f64", True)}


def _mix_int(x: int) -> int:
    x &= MASK64
    x = ((x ^ (x >> 30)) * M1) & MASK64
    x = ((x ^ (x >> 27)) * M2) & MASK64
    return x ^ (x >> 31)


def stream_key(seed: int, *tags) -> int:
    """64-bit key for a named stream, e.g. stream_key(seed, 'cfg2', 's', 16, 'A')."""
    h = 0x6A09E667F3BCC909
    for t in tags:
        for byte in str(t).encode():
            h = _mix_int(h ^ byte)
        h = _mix_int(h ^ 0xFF)
    return _mix_int((seed & MASK64) ^ h)


def _signed(x: int) -> int:
    return x - (1 << 64) if x >= (1 << 63) else x


# ----------------------------------------------------------- numpy (host) path
def raw_u64_numpy(key: int, start: int, count: int) -> np.ndarray:
    e = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.uint64(key) + e * np.uint64(GAMMA)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(M1)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(M2)
        x = x ^ (x >> np.uint64(31))
    return x


def _to_values_numpy(x: np.ndarray, prec: str, dist: str) -> np.ndarray:
    if dist == "int":
        return ((x >> np.uint64(32)) % np.uint64(9)).astype(np.int64).astype(np.float64) - 4.0
    if prec == "f64":
        return (x >> np.uint64(11)).astype(np.float64) * 2.0**-52 - 1.0
    return (x >> np.uint64(40)).astype(np.float64) * 2.0**-23 - 1.0


def values_numpy(kind: str, key: int, start: int, count: int, dist: str = "uniform") -> np.ndarray:
    """`count` scalars of `kind` (complex: 2 reals each, re then im) from element
    `start` of the stream."""
    prec, cplx = _KIND_DT[kind]
    nreal = count * (2 if cplx else 1)
    v = _to_values_numpy(raw_u64_numpy(key, start * (2 if cplx else 1), nreal), prec, dist)
    if prec == "f32":
        v = v.astype(np.float32)
    if cplx:
        v = v.view(np.complex64 if prec == "f32" else np.complex128)
    return v


# ------------------------------------------------------------ torch (any device)
def _lsr(t, s: int):
    """Logical shift right of an int64 tensor holding uint64 bits."""
    return (t >> s) & ((1 << (64 - s)) - 1)


def raw_u64_torch(key: int, start: int, count: int, device):
    import torch

    e = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    x = e * _signed(GAMMA) + _signed(key)
    x = (x ^ _lsr(x, 30)) * _signed(M1)
    x = (x ^ _lsr(x, 27)) * _signed(M2)
    return x ^ _lsr(x, 31)


def values_torch(kind: str, key: int, start: int, count: int, device, dist: str = "uniform",
                 chunk: int = 1 << 26):
    """Same values as values_numpy, produced by torch int64 ops on `device`
    (chunked so very large batches do not need 8-byte temporaries for all of it)."""
    import torch

    prec, cplx = _KIND_DT[kind]
    per = 2 if cplx else 1
    nreal = count * per
    rdt = torch.float32 if prec == "f32" else torch.float64
    out = torch.empty(nreal, dtype=rdt, device=device)
    s0 = start * per
    for c0 in range(0, nreal, chunk):
        c1 = min(nreal, c0 + chunk)
        x = raw_u64_torch(key, s0 + c0, c1 - c0, device)
        if dist == "int":
            v = torch.remainder(_lsr(x, 32), 9).to(torch.float64) - 4.0
        elif prec == "f64":
            v = _lsr(x, 11).to(torch.float64) * 2.0**-52 - 1.0
        else:
            v = _lsr(x, 40).to(torch.float64) * 2.0**-23 - 1.0
        out[c0:c1] = v.to(rdt)
    if cplx:
        out = torch.view_as_complex(out.view(-1, 2))
    return out


# ------------------------------------------------------------------- scalars
def scalar(kind: str, key: int, index: int = 0, dist: str = "uniform"):
    """One alpha/beta draw: U[-1,1) per component, rejecting |component| < 0.1
    and exact 0 / +-1, so the general epilogue is exercised.
    Deterministic: rejection walks the stream from element 2*index*64."""
    prec, cplx = _KIND_DT[kind]
    need = 2 if cplx else 1
    got = []
    e = index * 128
    while len(got) < need:
        x = np.array([raw_u64_numpy(key, e, 1)[0]], dtype=np.uint64)
        v = float(_to_values_numpy(x, prec, dist)[0])
        if prec == "f32":
            v = float(np.float32(v))
        e += 1
        if dist == "int":
            if v != 0:
                got.append(v)
            continue
        if abs(v) >= 0.1 and v not in (0.0, 1.0, -1.0):
            got.append(v)
    return complex(got[0], got[1]) if cplx else got[0]


def chunk_ranges(n: int, parts: int):
    """Balanced contiguous partition of [0, n) into min(parts, n) ranges; earlier
    ranges take the remainder.  Used to shard a batch over ranks."""
    if n <= 0:
        return []
    parts = max(1, min(parts, n))
    q, r = divmod(n, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + q + (1 if i < r else 0)
        out.append((lo, hi))
        lo = hi
    return out
