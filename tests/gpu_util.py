"""GPU-side test plumbing: upload seeded host batches, call the library through
the C ABI, download results.  No arithmetic of the method here."""
from __future__ import annotations

import numpy as np

import oracle
import paper_1304_7053_b200 as tx
from helpers import TOL, WIDE, Operand, denominators, max_rel_err

TORCH_DT = None


def torch_dtype(kind):
    import torch

    return {"s": torch.float32, "d": torch.float64, "c": torch.complex64, "z": torch.complex128}[kind]


def to_dev(op: Operand, extra=0):
    """Device copy of op.buf with `extra` leading elements so the base can be
    misaligned on purpose.  Returns (tensor, element offset of op.buf[0])."""
    import torch

    t = torch.from_numpy(op.buf.copy()).to("cuda")
    if extra:
        t2 = torch.zeros(t.numel() + extra, dtype=t.dtype, device="cuda")
        t2[extra:] = t
        return t2, extra
    return t, 0


def run_lib(kind, ta, tb, m, n, k, alpha, beta, A: Operand, B: Operand, C: Operand, misalign=0,
            stream=None):
    """Strided call on device copies; returns (status, C buffer as numpy, path)."""
    import torch

    dA, oa = to_dev(A, misalign)
    dB, ob = to_dev(B, misalign)
    dC, oc = to_dev(C, misalign)
    es = dA.element_size()
    rc = tx.tx_gemm_batched(kind, ta, tb, m, n, k, alpha, dA.data_ptr() + (oa + A.off) * es, A.ld,
                            A.ld2, dB.data_ptr() + (ob + B.off) * es, B.ld, B.ld2, beta,
                            dC.data_ptr() + (oc + C.off) * es, C.ld, C.ld2, C.batch, stream)
    path = tx.last_path()
    torch.cuda.synchronize()
    return rc, dC[oc:].cpu().numpy(), path


def run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C):
    Cref = C.buf.copy()
    rc = oracle.gemm_batched(kind, ta, tb, m, n, k, alpha, A.buf, A.ld, A.ld2, B.buf, B.ld, B.ld2,
                             beta, Cref, C.ld, C.ld2, C.batch, A.off, B.off, C.off)
    assert rc == 0
    return Cref


def check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got_buf, ref_buf):
    """Element-wise parity within the north-star tolerance, normalised by
    |alpha| sum |op(A)||op(B)| + |beta||C0|."""
    C0 = C.dense()
    den = denominators(kind, ta, tb, alpha, beta, A, B, C0)
    got = C.dense(got_buf)
    ref = C.dense(ref_buf)
    err = max_rel_err(kind, got, ref, den)
    assert err <= TOL[kind], f"max rel err {err:.3e} > {TOL[kind]} ({kind} {ta}{tb} {m}x{n}x{k})"
    return err
