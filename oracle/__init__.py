"""Parity oracle for the batched small-matrix GEMM -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1304_7053_b200`` never imports it, and this package imports nothing from
the product.  The arithmetic lives in ``oracle.c`` (plain C, see its header for
the definition it follows: PAPER.md:251-255 [§2 Eq. (1)], PAPER.md:360-362 [§5],
PAPER.md:454-466 [§6], PAPER.md:567-572 [§8]); this module only marshals numpy
buffers into that C library through ctypes.

Every function here is pinned by ``tests/test_oracle_pins.py``; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]

KINDS = ("s", "d", "c", "z")
NP_DTYPE = {"s": np.float32, "d": np.float64, "c": np.complex64, "z": np.complex128}
_REAL = {"s": ctypes.c_float, "d": ctypes.c_double}


class _CF(ctypes.Structure):
    _fields_ = [("re", ctypes.c_float), ("im", ctypes.c_float)]


class _CD(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


_SCALAR = {"s": ctypes.c_float, "d": ctypes.c_double, "c": _CF, "z": _CD}

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -ffp-contract=off: no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    """The oracle library.  ORACLE_LIB=<path> loads another build of oracle.c instead
    (used only by tests/test_oracle_mutations.py to run the pins against deliberately
    broken variants)."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("ORACLE_LIB")
            if not path:
                build()
                path = _LIB
            L = ctypes.CDLL(path)
            vp, c_int, c_ll, c_char = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_char
            for k in KINDS:
                f = getattr(L, f"oracle_gemm_batched_{k}")
                f.argtypes = [c_char, c_char, c_int, c_int, c_int, vp, vp, c_int, c_ll, vp, c_int,
                              c_ll, vp, vp, c_int, c_ll, c_int]
                f.restype = c_int
                g = getattr(L, f"oracle_gemm_batched_ptr_{k}")
                g.argtypes = [c_char, c_char, c_int, c_int, c_int, vp, vp, c_int, vp, c_int, vp, vp,
                              c_int, c_int]
                g.restype = c_int
            _lib = L
    return _lib


def _scalar(kind: str, v):
    v = complex(v)
    if kind in ("s", "d"):
        if v.imag != 0:
            raise ValueError("complex scalar for a real kind")
        return _SCALAR[kind](v.real)
    return _SCALAR[kind](v.real, v.imag)


def _ptr(arr, offset=0):
    if arr is None:
        return None
    assert isinstance(arr, np.ndarray) and arr.flags.c_contiguous
    return arr.ctypes.data + int(offset) * arr.itemsize


def _op(c):
    return c.encode() if isinstance(c, str) else bytes([c])


def gemm_batched(kind, transa, transb, m, n, k, alpha, A, lda, lda2, B, ldb, ldb2, beta, C,
                 ldc, ldc2, batch, a_off=0, b_off=0, c_off=0, alpha_ptr=True, beta_ptr=True):
    """Strided (uniform, second leading dimension) batch, in place on numpy C.

    ``A``/``B``/``C`` are flat numpy buffers of the kind's dtype (or None); the
    matrices start at element offsets ``a_off``/``b_off``/``c_off``.  Returns the
    status code (0 or -argpos).  ``alpha_ptr=False`` passes a NULL alpha.
    """
    L = lib()
    a = _scalar(kind, alpha)
    b = _scalar(kind, beta)
    return getattr(L, f"oracle_gemm_batched_{kind}")(
        _op(transa), _op(transb), m, n, k,
        ctypes.addressof(a) if alpha_ptr else None,
        _ptr(A, a_off), lda, lda2, _ptr(B, b_off), ldb, ldb2,
        ctypes.addressof(b) if beta_ptr else None,
        _ptr(C, c_off), ldc, ldc2, batch)


def gemm_batched_ptr(kind, transa, transb, m, n, k, alpha, A, a_offs, lda, B, b_offs, ldb, beta,
                     C, c_offs, ldc, batch, alpha_ptr=True, beta_ptr=True, null_arrays=()):
    """Pointer-array batch: matrix p of X starts at X[x_offs[p]] (the paper's nounif /
    cuBLAS-like interface)."""
    L = lib()
    a = _scalar(kind, alpha)
    b = _scalar(kind, beta)

    def arr(buf, offs, name):
        if name in null_arrays or buf is None:
            return None, None
        offs = np.asarray(offs, dtype=np.int64)
        ptrs = (ctypes.c_void_p * max(1, len(offs)))(*[_ptr(buf, o) for o in offs])
        return ptrs, ctypes.addressof(ptrs)

    ka, pa = arr(A, a_offs, "A")
    kb, pb = arr(B, b_offs, "B")
    kc, pc = arr(C, c_offs, "C")
    rc = getattr(L, f"oracle_gemm_batched_ptr_{kind}")(
        _op(transa), _op(transb), m, n, k, ctypes.addressof(a) if alpha_ptr else None,
        pa, lda, pb, ldb, ctypes.addressof(b) if beta_ptr else None, pc, ldc, batch)
    del ka, kb, kc
    return rc
