"""Shared test utilities: seeded batches in strided / pointer layouts, dense op()
views for error denominators, and the parity check of DESIGN.md §Parity.

Nothing here computes a GEMM: reference values come from oracle/ only."""
from __future__ import annotations

import numpy as np

import txinputs

NP = {"s": np.float32, "d": np.float64, "c": np.complex64, "z": np.complex128}
WIDE = {"s": np.float64, "d": np.float64, "c": np.complex128, "z": np.complex128}
TOL = {"s": 1e-5, "c": 1e-5, "d": 1e-13, "z": 1e-13}  # BASELINE.json north_star
TINY = {"s": np.finfo(np.float32).tiny, "c": np.finfo(np.float32).tiny,
        "d": np.finfo(np.float64).tiny, "z": np.finfo(np.float64).tiny}
OPS_REAL = ("N", "T")
OPS_CPLX = ("N", "T", "C")


def stored_shape(op, rows_op, cols_op):
    """Stored (rows, cols) of X when op(X) is rows_op x cols_op (R8)."""
    return (rows_op, cols_op) if op in "nN" else (cols_op, rows_op)


class Operand:
    """One batch operand in the strided layout: flat buffer + (off, ld, ld2)."""

    def __init__(self, kind, rows, cols, batch, key, pad_ld=0, pad_ld2=0, dist="uniform",
                 off=0, sentinel=None):
        self.kind, self.rows, self.cols, self.batch = kind, rows, cols, batch
        self.ld = max(1, rows + pad_ld)
        self.ld2 = self.ld * cols + pad_ld2
        self.off = off
        self.size = off + (self.ld2 * (batch - 1) + self.ld * (cols - 1) + rows if batch and rows and cols else 0)
        n = max(self.size, 1)
        if sentinel is None:
            self.buf = txinputs.values_numpy(kind, key, 0, n, dist).copy()
        else:
            self.buf = np.full(n, sentinel, dtype=NP[kind])
            vals = txinputs.values_numpy(kind, key, 0, n, dist)
            m = self.mask()
            self.buf[m] = vals[m]

    def index(self, p, i, j):
        return self.off + i + self.ld * j + self.ld2 * p

    def mask(self):
        """Boolean mask of the buffer entries that belong to a matrix."""
        m = np.zeros(max(self.size, 1), dtype=bool)
        if self.size:
            p = np.arange(self.batch)[:, None, None]
            i = np.arange(self.rows)[None, :, None]
            j = np.arange(self.cols)[None, None, :]
            m[(self.off + i + self.ld * j + self.ld2 * p).ravel()] = True
        return m

    def dense(self, buf=None):
        """(batch, rows, cols) view of the stored matrices (a copy)."""
        b = self.buf if buf is None else buf
        p = np.arange(self.batch)[:, None, None]
        i = np.arange(self.rows)[None, :, None]
        j = np.arange(self.cols)[None, None, :]
        return b[self.off + i + self.ld * j + self.ld2 * p]

    def offsets(self):
        return self.off + self.ld2 * np.arange(self.batch, dtype=np.int64)


def op_dense(X: np.ndarray, op: str) -> np.ndarray:
    if op in "nN":
        return X
    Y = np.swapaxes(X, 1, 2)
    return np.conj(Y) if op in "cC" else Y


def denominators(kind, transa, transb, alpha, beta, A: Operand, B: Operand, C0: np.ndarray):
    """den_ij = |alpha| * sum_l |op(A)_il| |op(B)_lj| + |beta| |C0_ij|."""
    a = np.abs(op_dense(A.dense().astype(WIDE[kind]), transa))
    b = np.abs(op_dense(B.dense().astype(WIDE[kind]), transb))
    d = abs(alpha) * np.einsum("pil,plj->pij", a, b)
    if beta != 0:
        d = d + abs(beta) * np.abs(C0.astype(WIDE[kind]))
    return d


def max_rel_err(kind, got, ref, den):
    got = np.asarray(got).astype(WIDE[kind])
    ref = np.asarray(ref).astype(WIDE[kind])
    diff = np.abs(got - ref)
    exact_needed = den == 0
    if np.any(exact_needed & (diff != 0)):
        return np.inf
    with np.errstate(divide="ignore", invalid="ignore"):
        e = np.where(exact_needed, 0.0, diff / np.maximum(den, TINY[kind]))
    if np.any(np.isnan(e)):
        return np.inf
    return float(e.max()) if e.size else 0.0


def random_case(kind, m, n, k, batch, transa="N", transb="N", seed=1, tag="case", pad=(0, 0),
                dist="uniform", c_sentinel=None):
    key = lambda name: txinputs.stream_key(seed, tag, kind, m, n, k, transa, transb, name)
    ra, ca = stored_shape(transa, m, k)
    rb, cb = stored_shape(transb, k, n)
    A = Operand(kind, ra, ca, batch, key("A"), pad[0], pad[1], dist)
    B = Operand(kind, rb, cb, batch, key("B"), pad[0], pad[1], dist)
    C = Operand(kind, m, n, batch, key("C"), pad[0], pad[1], dist, sentinel=c_sentinel)
    return A, B, C


def dense_at(buf, offs, rows, cols, ld):
    """(batch, rows, cols) copy of the matrices starting at element offsets offs
    (pointer-array layouts), column-major with leading dimension ld."""
    offs = np.asarray(offs, dtype=np.int64)[:, None, None]
    i = np.arange(rows)[None, :, None]
    j = np.arange(cols)[None, None, :]
    return buf[offs + i + ld * j]


def denominators_dense(kind, transa, transb, alpha, beta, Ad, Bd, C0d):
    """Element-wise |alpha| sum_l |op(A)_il||op(B)_lj| + |beta||C0_ij| from dense stored
    (batch, rows, cols) arrays."""
    a = np.abs(op_dense(np.asarray(Ad).astype(WIDE[kind]), transa))
    b = np.abs(op_dense(np.asarray(Bd).astype(WIDE[kind]), transb))
    d = abs(alpha) * np.einsum("pil,plj->pij", a, b)
    if beta != 0:
        d = d + abs(beta) * np.abs(np.asarray(C0d).astype(WIDE[kind]))
    return d
