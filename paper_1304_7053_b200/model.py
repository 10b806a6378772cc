"""Work model of one batched GEMM call (host logic, no arithmetic of the method).

flops: the paper's convention: 2 m n k per real pair and
8 m n k per complex pair, for all alpha, beta and op ("3M" not used); the paper
states it for square sizes as 2m^3 / 8m^3.

bytes: the ALGORITHMIC bytes the method must move through HBM:
A and B are read when alpha != 0 and k > 0, C is read only when beta != 0 and
always written (the beta == 0 path never reads C).  Padding
is not counted; the pointer layout adds 8 bytes per array entry read.
"""
from __future__ import annotations

ESIZE = {"s": 4, "d": 8, "c": 8, "z": 16}
CPLX = {"s": False, "d": False, "c": True, "z": True}


def flops(kind: str, m: int, n: int, k: int, batch: int) -> int:
    return (8 if CPLX[kind] else 2) * m * n * k * batch


def bytes_moved(kind: str, m: int, n: int, k: int, batch: int, alpha_nonzero: bool = True,
                beta_nonzero: bool = False, pointer_arrays: bool = False,
                shared_a: bool = False, shared_b: bool = False) -> int:
    """shared_a / shared_b: fixed-operand batch (ld2 = 0), the shared
    matrix is read once for the whole batch."""
    s = ESIZE[kind]
    reads_ab = alpha_nonzero and k > 0
    a = 0 if (shared_a or not reads_ab) else m * k
    b = 0 if (shared_b or not reads_ab) else k * n
    per = s * (a + b + m * n * (2 if beta_nonzero else 1))
    if pointer_arrays:
        per += 8 * ((2 if reads_ab else 0) + 1)
    once = s * ((m * k if shared_a and reads_ab else 0) + (k * n if shared_b and reads_ab else 0))
    return per * batch + (once if batch else 0)


def footprint(kind: str, m: int, n: int, k: int, batch: int) -> int:
    """Bytes resident for packed A, B and C (PAPER.md:588-591's 1.23 GB example)."""
    return ESIZE[kind] * (m * k + k * n + m * n) * batch
