"""Small cases for compute-sanitizer (SURVEY §4 tier T1s).  Exercises the bulk
(TMA + mbarrier) kernels, the gather / pointer kernels (JIT) and the scale kernel.
With --uninit-c, C is allocated with cudaMalloc and never written before the
beta == 0 call: initcheck then proves the beta == 0 path never reads C."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1304_7053_b200 as tx  # noqa: E402
import txinputs  # noqa: E402


def main():
    uninit = "--uninit-c" in sys.argv
    # d16 / z16 with op(A) = T: the TMA tensor-copy (ASW) instances, ragged last box
    for kind, n, batch in (("s", 16, 3000), ("d", 5, 1001), ("c", 8, 517), ("z", 3, 999),
                           ("d", 16, 37), ("z", 16, 21)):
        ta0 = "T" if n == 16 and kind in "dz" else "N"
        e = n * n
        A = txinputs.values_torch(kind, 1, 0, e * batch, "cuda")
        B = txinputs.values_torch(kind, 2, 0, e * batch, "cuda")
        C = torch.empty(e * batch, dtype=A.dtype, device="cuda")  # uninitialised
        assert tx.tx_gemm_batched(kind, ta0, "T", n, n, n, 1.0, A, n, e, B, n, e, 0.0, C, n, e,
                                  batch) == 0
        if not uninit:
            assert tx.tx_gemm_batched(kind, "T", "N", n, n, n, 0.5, A, n, e, B, n, e, 0.25, C, n, e,
                                      batch) == 0
            assert tx.tx_gemm_batched(kind, "N", "N", n, n, n, 0.0, A, n, e, B, n, e, 0.5, C, n, e,
                                      batch) == 0
            # pointer arrays and a padded layout (gather kernels)
            es = A.element_size()
            idx = torch.arange(batch, device="cuda")
            pa, pb, pc = (X.data_ptr() + idx * (e * es) for X in (A, B, C))
            assert tx.tx_gemm_batched_ptr(kind, "N", "N", n, n, n, 0.5, pa, n, pb, n, 0.25, pc, n,
                                          batch) == 0
            Cp = torch.zeros((e + 3) * batch, dtype=A.dtype, device="cuda")
            assert tx.tx_gemm_batched(kind, "N", "N", n, n, n, 1.0, A, n, e, B, n, e, 0.5, Cp, n,
                                      e + 3, batch) == 0
    # runtime-specialised non-square instances with swizzled (TMA tensor) A / B tiles
    # and the swizzled gather placement (pointer arrays), ragged batches
    for kind, (m, n, k), ta, tb, batch in (("z", (1, 16, 16), "N", "N", 23),
                                           ("c", (16, 3, 16), "T", "T", 19),
                                           ("d", (5, 6, 16), "T", "N", 31)):
        A = txinputs.values_torch(kind, 4, 0, m * k * batch, "cuda")
        B = txinputs.values_torch(kind, 5, 0, k * n * batch, "cuda")
        C = txinputs.values_torch(kind, 6, 0, m * n * batch, "cuda")
        lda = m if ta == "N" else k
        ldb = k if tb == "N" else n
        for beta in (0.0, 0.5):
            assert tx.tx_gemm_batched(kind, ta, tb, m, n, k, 1.0, A, lda, m * k, B, ldb, k * n, beta,
                                      C, m, m * n, batch) == 0
        if not uninit:
            es = A.element_size()
            idx = torch.arange(batch, device="cuda")
            pa, pb, pc = (X.data_ptr() + idx * (s * es) for X, s in ((A, m * k), (B, k * n), (C, m * n)))
            assert tx.tx_gemm_batched_ptr(kind, ta, tb, m, n, k, 0.5, pa, lda, pb, ldb, 0.25, pc, m,
                                          batch) == 0
    # pointer arrays of 16x16 matrices through bulk_ptr (decoupled ring for d / z general,
    # per-tile barrier for s general and c beta = 0) with the grid capped at 2 CTAs so every
    # CTA cycles its stages many times (mbarrier phase flips, empty-barrier waits)
    if not uninit:
        prev = tx.set_max_ctas(2)
        try:
            for kind, beta in (("d", 0.25), ("z", 0.25), ("s", 0.25), ("c", 0.0)):
                n, batch = 16, 96
                e = n * n
                A = txinputs.values_torch(kind, 7, 0, e * batch, "cuda")
                B = txinputs.values_torch(kind, 8, 0, e * batch, "cuda")
                C = txinputs.values_torch(kind, 9, 0, e * batch, "cuda")
                es = A.element_size()
                idx = torch.randperm(batch, generator=torch.Generator().manual_seed(5)).cuda()
                pa, pb, pc = (X.data_ptr() + idx * (e * es) for X in (A, B, C))
                assert tx.tx_gemm_batched_ptr(kind, "N", "N", n, n, n, 0.5, pa, n, pb, n, beta, pc,
                                              n, batch) == 0
        finally:
            tx.set_max_ctas(prev)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
