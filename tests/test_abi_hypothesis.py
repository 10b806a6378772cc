"""Property test (SURVEY §4 tier T0): for random argument vectors, the library's host
validation returns exactly the oracle's code whenever the oracle rejects the vector.
Valid vectors are not sent to the library (they would launch kernels on fake pointers)."""
import ctypes

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
import paper_1304_7053_b200 as tx

FAKE = 1 << 40
OPS = st.sampled_from(list("nNtTcCxq "))


@settings(max_examples=400, deadline=None)
@given(kind=st.sampled_from("sdcz"), ta=OPS, tb=OPS, m=st.integers(-2, 66), n=st.integers(-2, 66),
       k=st.integers(-2, 66), lda=st.integers(-1, 68), ldb=st.integers(-1, 68),
       ldc=st.integers(-1, 68), lda2=st.integers(-3, 1200), ldb2=st.integers(-3, 1200),
       ldc2=st.integers(-3, 1200), batch=st.integers(-2, 5), alpha=st.sampled_from([0.0, 1.0, 2.5]),
       beta=st.sampled_from([0.0, 1.0, -0.5]), a_null=st.booleans(), b_null=st.booleans(),
       c_null=st.booleans(), alpha_ptr=st.booleans(), beta_ptr=st.booleans(),
       c_off=st.integers(0, 4000))
def test_validation_equivalence(kind, ta, tb, m, n, k, lda, ldb, ldc, lda2, ldb2, ldc2, batch, alpha,
                                beta, a_null, b_null, c_null, alpha_ptr, beta_ptr, c_off):
    es = {"s": 4, "d": 8, "c": 8, "z": 16}[kind]
    base = np.zeros(40000, dtype=oracle.NP_DTYPE[kind])
    offs = {"A": 0, "B": 12000, "C": 24000 - c_off}

    def host(name, null):
        return None if null else base.ctypes.data + offs[name] * es

    def fake(name, null):
        return None if null else FAKE + offs[name] * es

    L = oracle.lib()
    a_s, b_s = oracle._scalar(kind, alpha), oracle._scalar(kind, beta)
    want = getattr(L, f"oracle_gemm_batched_{kind}")(
        ta.encode(), tb.encode(), m, n, k, ctypes.addressof(a_s) if alpha_ptr else None,
        host("A", a_null), lda, lda2, host("B", b_null), ldb, ldb2,
        ctypes.addressof(b_s) if beta_ptr else None, host("C", c_null), ldc, ldc2, batch)
    if want == 0:
        return  # valid: the library would launch on fake pointers
    got = tx.tx_gemm_batched(kind, ta, tb, m, n, k, alpha, fake("A", a_null), lda, lda2,
                             fake("B", b_null), ldb, ldb2, beta, fake("C", c_null), ldc, ldc2,
                             batch, stream=0, alpha_ptr=alpha_ptr, beta_ptr=beta_ptr)
    assert got == want
