"""Pins for the CPU oracle (oracle/oracle.c) -- run with -m "not gpu".

Each test ties the oracle to something other than itself: values printed in the
paper/SPEC (tests/golden/), closed forms, invariants, a library routine (numpy
float64 einsum), or exact rational arithmetic (fractions) within the textbook
error bound |fl(x^T y) - x^T y| <= gamma_k sum|x||y|.  Together they fail on a
dropped term, a wrong sign, a wrong index or a transposed operand.
"""
from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import txinputs
from helpers import (NP, WIDE, Operand, denominators, max_rel_err, op_dense, random_case,
                     stored_shape)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U = {"s": 2.0**-24, "c": 2.0**-24, "d": 2.0**-53, "z": 2.0**-53}


def _vals(kind, lst):
    out = []
    for v in lst:
        if isinstance(v, list):
            out.append(complex(v[0], v[1]))
        elif v == "nan":
            out.append(complex("nan") if kind in "cz" else float("nan"))
        else:
            out.append(v)
    return np.array(out, dtype=NP[kind])


def _scal(v):
    return complex(v[0], v[1]) if isinstance(v, list) else v


def run_strided(kind, ta, tb, m, n, k, alpha, A, B, beta, C):
    return oracle.gemm_batched(kind, ta, tb, m, n, k, alpha, A.buf, A.ld, A.ld2, B.buf, B.ld,
                               B.ld2, beta, C.buf, C.ld, C.ld2, C.batch, A.off, B.off, C.off)


# ------------------------------------------------------------------ golden cases
HAND = json.load(open(os.path.join(GOLD, "hand_cases.json")))["cases"]


@pytest.mark.parametrize("case", HAND, ids=[c["name"] for c in HAND])
def test_hand_cases(case):
    for kind in case["kinds"]:
        A = _vals(kind, case["A"])
        B = _vals(kind, case["B"])
        C = _vals(kind, case["C0"])
        rc = oracle.gemm_batched(kind, case["transa"], case["transb"], case["m"], case["n"],
                                 case["k"], _scal(case["alpha"]), A, case["lda"], 0, B,
                                 case["ldb"], 0, _scal(case["beta"]), C, case["ldc"], 0, 1)
        assert rc == 0
        want = _vals(kind, case["C"])
        assert np.array_equal(C, want), (kind, C, want)


PAPER = json.load(open(os.path.join(GOLD, "paper_numbers.json")))


@pytest.mark.parametrize("ex", PAPER["element_offset"], ids=lambda e: str(e["offset"]))
def test_element_offset(ex):
    """X[i + ld*j + ld2*p]: a single 1 at the printed offset of A,
    B = I, must appear at (i, j) of matrix p of C and nowhere else."""
    base, ld, ld2, i, j, p = (ex[k] for k in ("base", "ld", "ld2", "i", "j", "p"))
    m, k = ld, (ld2 // ld)  # A is m x k, fully using ld and ld2
    batch = p + 1
    size = base + ld2 * (batch - 1) + ld * (k - 1) + m
    A = np.zeros(size, dtype=np.float64)
    A[ex["offset"]] = 1.0
    assert ex["offset"] == base + i + ld * j + ld2 * p
    Bm = np.eye(k).ravel(order="F")
    B = np.tile(Bm, batch)
    C = np.zeros(m * k * batch)
    rc = oracle.gemm_batched("d", "N", "N", m, k, k, 1.0, A, ld, ld2, B, k, k * k, 0.0, C, m,
                             m * k, batch, a_off=base)
    assert rc == 0
    nz = np.flatnonzero(C)
    assert list(nz) == [i + m * j + m * k * p]


# --------------------------------------------------------------- closed forms
def _int_case(kind, m, n, k, batch, ta="N", tb="N", tag="int"):
    return random_case(kind, m, n, k, batch, ta, tb, seed=3, tag=tag, dist="int")


@pytest.mark.parametrize("kind", "sdcz")
def test_identity_left_gives_B(kind):
    m = n = k = 7
    A, B, C = random_case(kind, m, n, k, 5, seed=4, tag="idl")
    A.buf[:] = np.tile(np.eye(m).ravel(order="F"), 5).astype(NP[kind])
    C.buf[:] = np.nan
    assert run_strided(kind, "N", "N", m, n, k, 1, A, B, 0, C) == 0
    assert np.array_equal(C.dense(), B.dense())


@pytest.mark.parametrize("kind", "sdcz")
def test_permutation_left_permutes_rows(kind):
    m = n = k = 6
    rng = np.random.default_rng(0)
    A, B, C = random_case(kind, m, n, k, 4, seed=5, tag="perm")
    perms = [rng.permutation(m) for _ in range(4)]
    D = np.zeros((4, m, k))
    for p, pi in enumerate(perms):
        D[p, np.arange(m), pi] = 1
    A.buf[:] = D.transpose(0, 2, 1).ravel().astype(NP[kind])
    assert run_strided(kind, "N", "N", m, n, k, 1, A, B, 0, C) == 0
    got = C.dense()
    Bd = B.dense()
    for p, pi in enumerate(perms):
        assert np.array_equal(got[p], Bd[p][pi])


@pytest.mark.parametrize("kind", "sdcz")
def test_zero_A_gives_beta_C(kind):
    m, n, k = 5, 4, 3
    A, B, C = _int_case(kind, m, n, k, 6)
    A.buf[:] = 0
    beta = txinputs.scalar(kind, 99, dist="int")
    C0 = C.dense().astype(WIDE[kind])
    assert run_strided(kind, "N", "N", m, n, k, 2, A, B, beta, C) == 0
    assert np.array_equal(C.dense().astype(WIDE[kind]), beta * C0)


@pytest.mark.parametrize("kind", "sdcz")
def test_alpha_zero_never_reads_AB(kind):
    m, n, k = 4, 5, 6
    A, B, C = _int_case(kind, m, n, k, 3)
    A.buf[:] = np.nan
    B.buf[:] = np.nan
    beta = txinputs.scalar(kind, 7, dist="int")
    C0 = C.dense().astype(WIDE[kind])
    assert run_strided(kind, "N", "N", m, n, k, 0, A, B, beta, C) == 0
    assert np.array_equal(C.dense().astype(WIDE[kind]), beta * C0)


@pytest.mark.parametrize("kind", "sdcz")
def test_beta_zero_never_reads_C(kind):
    m, n, k = 6, 6, 6
    A, B, C = random_case(kind, m, n, k, 3, seed=8, tag="b0")
    C.buf[:] = np.nan
    alpha = txinputs.scalar(kind, 11)
    assert run_strided(kind, "N", "N", m, n, k, alpha, A, B, 0, C) == 0
    assert np.all(np.isfinite(C.dense()))


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("ops", [("N", "N"), ("T", "C")])
def test_beta_zero_general_alpha_is_alpha_times_product(kind, ops):
    """beta = 0 with a general alpha: y = alpha*x and C is never read (R3,
    PAPER.md:436-466).  Integer inputs make every value exact, so C(alpha, 0) must equal
    alpha * C(1, 0) bitwise, where C(1, 0) is itself pinned by the hand cases; C starts
    as NaN.  Fails for `y = x` (alpha dropped) and for any read of C."""
    ta, tb = ops
    m, n, k, batch = 7, 5, 9, 6
    A, B, C = random_case(kind, m, n, k, batch, ta, tb, seed=31, tag="a3b0", dist="int")
    C.buf[:] = np.nan
    C1 = Operand(kind, m, n, batch, 0)
    C1.buf[:] = np.nan
    alpha = 3 if kind in "sd" else complex(2, -1)
    assert run_strided(kind, ta, tb, m, n, k, 1, A, B, 0, C1) == 0
    assert run_strided(kind, ta, tb, m, n, k, alpha, A, B, 0, C) == 0
    got = C.dense().astype(WIDE[kind])
    assert np.all(np.isfinite(got))
    assert np.array_equal(got, alpha * C1.dense().astype(WIDE[kind]))
    assert np.any(got != C1.dense())  # alpha really changed the values


@pytest.mark.parametrize("kind", "sdcz")
def test_validation_misaligned_pointers(kind):
    """A, B, C not aligned to the element size -> -7 / -10 / -14 (R21);
    pointer arrays not 8-byte aligned -> -7 / -9 / -12."""
    import ctypes

    es = {"s": 4, "d": 8, "c": 8, "z": 16}[kind]
    L = oracle.lib()
    buf = np.zeros(4096, dtype=np.uint8)
    base = (buf.ctypes.data + 63) // 64 * 64
    A, B, C = base, base + 1024, base + 2048
    a = oracle._scalar(kind, 1.0)
    b = oracle._scalar(kind, 0.0)
    f = getattr(L, f"oracle_gemm_batched_{kind}")

    def call(pa, pb, pc):
        return f(b"N", b"N", 2, 2, 2, ctypes.addressof(a), pa, 2, 4, pb, 2, 4, ctypes.addressof(b),
                 pc, 2, 4, 2)

    assert call(A, B, C) == 0
    for off in sorted({1, 2, es // 2, es - 1} - {0}):
        assert call(A + off, B, C) == -7
        assert call(A, B + off, C) == -10
        assert call(A, B, C + off) == -14
    g = getattr(L, f"oracle_gemm_batched_ptr_{kind}")
    ptrs = (ctypes.c_void_p * 8)(A, A, B, B, C, C, 0, 0)
    pa = ctypes.addressof(ptrs)

    def callp(x, y, z):
        return g(b"N", b"N", 2, 2, 2, ctypes.addressof(a), x, 2, y, 2, ctypes.addressof(b), z, 2, 1)

    assert callp(pa, pa + 16, pa + 32) == 0
    assert callp(pa + 4, pa + 16, pa + 32) == -7
    assert callp(pa, pa + 12, pa + 32) == -9
    assert callp(pa, pa + 16, pa + 36) == -12


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("k", [0, 5])
def test_alpha0_or_k0_with_beta1_is_untouched(kind, k):
    m, n = 3, 4
    A, B, C = random_case(kind, m, n, max(k, 1), 4, seed=9, tag="q")
    A.buf[:] = np.nan
    C.buf[0] = np.nan
    before = C.buf.copy()
    alpha = 0 if k else 1.5
    assert run_strided(kind, "N", "N", m, n, k, alpha, A, B, 1, C) == 0
    assert np.array_equal(C.buf.view(np.uint8), before.view(np.uint8))


@pytest.mark.parametrize("kind", "sdcz")
def test_k0_scales_C(kind):
    m, n = 5, 3
    A, B, C = _int_case(kind, m, n, 1, 4)
    beta = txinputs.scalar(kind, 12, dist="int")
    C0 = C.dense().astype(WIDE[kind])
    assert run_strided(kind, "N", "N", m, n, 0, 3, A, B, beta, C) == 0
    assert np.array_equal(C.dense().astype(WIDE[kind]), beta * C0)


# ----------------------------------------------------------------- invariants
@pytest.mark.parametrize("kind", "sdcz")
def test_transpose_rule_bitwise(kind):
    """(op(A)op(B))^T = op(B)^T op(A)^T: gemm('T','T', n,m,k, B, A) is the transpose of
    gemm('N','N', m,n,k, A, B), bitwise (same products, commutative IEEE x and 2-term +)."""
    m, n, k = 5, 7, 9
    A, B, C = random_case(kind, m, n, k, 6, seed=13, tag="tr")
    assert run_strided(kind, "N", "N", m, n, k, 1, A, B, 0, C) == 0
    Ct = Operand(kind, n, m, 6, 1)
    assert oracle.gemm_batched(kind, "T", "T", n, m, k, 1, B.buf, B.ld, B.ld2, A.buf, A.ld,
                               A.ld2, 0, Ct.buf, Ct.ld, Ct.ld2, 6) == 0
    assert np.array_equal(Ct.dense(), np.swapaxes(C.dense(), 1, 2))


@pytest.mark.parametrize("kind", "cz")
def test_hermitian_rule(kind):
    """(AB)^H = B^H A^H: gemm('C','C', n,m,k, B, A) = conj(gemm('N','N', m,n,k, A, B))^T."""
    m, n, k = 4, 6, 5
    A, B, C = random_case(kind, m, n, k, 5, seed=14, tag="h")
    assert run_strided(kind, "N", "N", m, n, k, 1, A, B, 0, C) == 0
    Ch = Operand(kind, n, m, 5, 1)
    assert oracle.gemm_batched(kind, "C", "C", n, m, k, 1, B.buf, B.ld, B.ld2, A.buf, A.ld,
                               A.ld2, 0, Ch.buf, Ch.ld, Ch.ld2, 5) == 0
    assert np.array_equal(Ch.dense(), np.conj(np.swapaxes(C.dense(), 1, 2)))


@pytest.mark.parametrize("kind", "sd")
def test_real_conj_equals_transpose(kind):
    """'C' on a real type is 'T' (PAPER.md:491-499 identity functor), bitwise."""
    m, n, k = 6, 5, 4
    A, B, C1 = random_case(kind, m, n, k, 3, "T", "T", seed=15, tag="rc")
    C2 = Operand(kind, m, n, 3, 77)
    C2.buf[:] = C1.buf
    alpha, beta = txinputs.scalar(kind, 1), txinputs.scalar(kind, 2)
    assert run_strided(kind, "T", "T", m, n, k, alpha, A, B, beta, C1) == 0
    assert run_strided(kind, "C", "c", m, n, k, alpha, A, B, beta, C2) == 0
    assert np.array_equal(C1.buf.view(np.uint8), C2.buf.view(np.uint8))


@pytest.mark.parametrize("kind", "sdcz")
def test_padded_equals_packed_and_pads_untouched(kind):
    m, n, k, batch = 5, 6, 7, 9
    Ap, Bp, Cp = random_case(kind, m, n, k, batch, "T", "N", seed=16, tag="pad")
    Aq, Bq, Cq = random_case(kind, m, n, k, batch, "T", "N", seed=16, tag="pad", pad=(3, 7),
                             c_sentinel=-7.25)
    # same matrix values in both layouts
    for src, dst in ((Ap, Aq), (Bp, Bq), (Cp, Cq)):
        idx = dst.index(np.arange(batch)[:, None, None], np.arange(dst.rows)[None, :, None],
                        np.arange(dst.cols)[None, None, :])
        dst.buf[idx] = src.dense()
    pad_before = Cq.buf[~Cq.mask()].copy()
    alpha, beta = txinputs.scalar(kind, 3), txinputs.scalar(kind, 4)
    assert run_strided(kind, "T", "N", m, n, k, alpha, Ap, Bp, beta, Cp) == 0
    assert run_strided(kind, "T", "N", m, n, k, alpha, Aq, Bq, beta, Cq) == 0
    assert np.array_equal(Cq.dense(), Cp.dense())
    assert np.array_equal(Cq.buf[~Cq.mask()].view(np.uint8), pad_before.view(np.uint8))


@pytest.mark.parametrize("kind", "sdcz")
def test_pointer_equals_strided_and_permutes(kind):
    """Pointer interface over as_handles(strided) == strided, bitwise;
    permuted pointers give permuted results."""
    m, n, k, batch = 6, 4, 5, 11
    A, B, C = random_case(kind, m, n, k, batch, "N", "C" if kind in "cz" else "T", seed=17,
                          tag="ptr", pad=(1, 2))
    tb = "C" if kind in "cz" else "T"
    C2 = C.buf.copy()
    alpha, beta = txinputs.scalar(kind, 5), txinputs.scalar(kind, 6)
    assert run_strided(kind, "N", tb, m, n, k, alpha, A, B, beta, C) == 0
    assert oracle.gemm_batched_ptr(kind, "N", tb, m, n, k, alpha, A.buf, A.offsets(), A.ld, B.buf,
                                   B.offsets(), B.ld, beta, C2, C.offsets(), C.ld, batch) == 0
    assert np.array_equal(C.buf.view(np.uint8), C2.view(np.uint8))
    perm = np.random.default_rng(1).permutation(batch)
    C3 = Operand(kind, m, n, batch, 0)
    C3.buf[:] = 0
    assert oracle.gemm_batched_ptr(kind, "N", tb, m, n, k, alpha, A.buf, A.offsets()[perm], A.ld,
                                   B.buf, B.offsets()[perm], B.ld, 0, C3.buf,
                                   C3.offsets(), C3.ld, batch) == 0
    C4 = Operand(kind, m, n, batch, 0)
    C4.buf[:] = 0
    assert run_strided(kind, "N", tb, m, n, k, alpha, A, B, 0, C4) == 0
    assert np.array_equal(C3.dense(), C4.dense()[perm])


# ------------------------------------------- library routine and exact arithmetic
def _gamma(kind, k):
    u = U[kind]
    kk = k + 4  # k-term sum + complex product/axpby roundings
    return kk * u / (1 - kk * u)


@pytest.mark.parametrize("kind", "sc")
@pytest.mark.parametrize("ops", [("N", "N"), ("T", "N"), ("N", "T"), ("C", "T"), ("T", "C")])
def test_single_precision_vs_numpy_float64(kind, ops):
    """fp32/c64 oracle vs numpy's float64 einsum (a library routine), within gamma_{k+4}."""
    ta, tb = ops
    if kind == "s" and "C" in ops:
        pytest.skip("C == T for real kinds (covered above)")
    m, n, k, batch = 16, 13, 16, 200
    A, B, C = random_case(kind, m, n, k, batch, ta, tb, seed=21, tag="np")
    alpha, beta = txinputs.scalar(kind, 31), txinputs.scalar(kind, 32)
    C0 = C.dense().astype(WIDE[kind])
    ref = alpha * np.einsum("pil,plj->pij", op_dense(A.dense().astype(WIDE[kind]), ta),
                            op_dense(B.dense().astype(WIDE[kind]), tb)) + beta * C0
    assert run_strided(kind, ta, tb, m, n, k, alpha, A, B, beta, C) == 0
    den = denominators(kind, ta, tb, alpha, beta, A, B, C0)
    err = max_rel_err(kind, C.dense(), ref, den)
    assert err <= _gamma(kind, k), err
    # and it is not trivially zero-error (the fp32 loop really rounds)
    assert err > 0


def _exact(kind, ta, tb, alpha, beta, A, B, C0):
    """Exact rational Eq. (1) on tiny inputs (Python Fractions; complex as (re, im))."""
    def F(x):
        return (Fraction(float(np.real(x))), Fraction(float(np.imag(x))))

    def mul(a, b):
        return (a[0] * b[0] - a[1] * b[1], a[0] * b[1] + a[1] * b[0])

    Ad, Bd = op_dense(A.dense(), ta), op_dense(B.dense(), tb)
    batch, m, k = Ad.shape
    n = Bd.shape[2]
    out = np.zeros((batch, m, n, 2), dtype=object)
    al, be = F(alpha), F(beta)
    for p in range(batch):
        for i in range(m):
            for j in range(n):
                s = (Fraction(0), Fraction(0))
                for l in range(k):
                    t = mul(F(Ad[p, i, l]), F(Bd[p, l, j]))
                    s = (s[0] + t[0], s[1] + t[1])
                y = mul(al, s)
                if beta != 0:
                    z = mul(be, F(C0[p, i, j]))
                    y = (y[0] + z[0], y[1] + z[1])
                out[p, i, j, 0], out[p, i, j, 1] = y
    return out


@pytest.mark.parametrize("kind", "dz")
@pytest.mark.parametrize("ops", [("N", "N"), ("T", "C"), ("C", "N")])
def test_double_precision_vs_exact_rationals(kind, ops):
    ta, tb = ops
    if kind == "d":
        ta, tb = ta.replace("C", "T"), tb.replace("C", "T")
    m, n, k, batch = 5, 4, 16, 3
    A, B, C = random_case(kind, m, n, k, batch, ta, tb, seed=22, tag="ex")
    alpha, beta = txinputs.scalar(kind, 41), txinputs.scalar(kind, 42)
    C0 = C.dense().copy()
    exact = _exact(kind, ta, tb, alpha, beta, A, B, C0)
    assert run_strided(kind, ta, tb, m, n, k, alpha, A, B, beta, C) == 0
    got = C.dense()
    den = denominators(kind, ta, tb, alpha, beta, A, B, C0)
    worst = 0.0
    for idx in np.ndindex(got.shape):
        g = complex(got[idx])
        er = abs(Fraction(g.real) - exact[idx + (0,)])
        ei = abs(Fraction(g.imag) - exact[idx + (1,)])
        e = float(max(er, ei))
        worst = max(worst, e / den[idx])
    assert worst <= _gamma(kind, k), worst


def test_dropped_term_would_fail_the_bound():
    """Sanity of the bound itself: removing the last k term from the numpy reference
    exceeds gamma_k by orders of magnitude, so the pins above detect such a bug."""
    kind, m, n, k = "s", 16, 16, 16
    A, B, C = random_case(kind, m, n, k, 50, seed=24, tag="drop")
    Ad = A.dense().astype(np.float64)
    Bd = B.dense().astype(np.float64)
    full = np.einsum("pil,plj->pij", Ad, Bd)
    short = np.einsum("pil,plj->pij", Ad[:, :, :-1], Bd[:, :-1, :])
    den = np.einsum("pil,plj->pij", np.abs(Ad), np.abs(Bd))
    assert (np.abs(full - short) / den).max() > 1e3 * _gamma(kind, k)


# ------------------------------------------------------------------ validation
def _args(**kw):
    d = dict(kind="d", ta="N", tb="N", m=4, n=4, k=4, alpha=1.0, lda=4, lda2=16, ldb=4, ldb2=16,
             beta=0.0, ldc=4, ldc2=16, batch=3, alpha_ptr=True, beta_ptr=True)
    d.update(kw)
    return d


VALIDATION = [
    ("ok", {}, 0),
    ("transa", {"ta": "x"}, -1),
    ("transb", {"tb": "Q"}, -2),
    ("m<0", {"m": -1}, -3),
    ("m>64", {"m": 65}, -3),
    ("n>64", {"n": 65}, -4),
    ("m=64 valid (real)", {"m": 64, "lda": 64, "ldc": 64, "ldc2": 256}, 0),
    ("m>32 complex", {"kind": "z", "m": 33, "lda": 33, "ldc": 33, "ldc2": 132}, -3),
    ("k>32 complex", {"kind": "c", "k": 33}, -5),
    ("m=17 valid", {"m": 17, "lda": 17, "ldc": 17, "ldc2": 68}, 0),
    ("k<0", {"k": -2}, -5),
    ("alpha NULL", {"alpha_ptr": False}, -6),
    ("beta NULL", {"beta_ptr": False}, -13),
    ("lda<m", {"lda": 3}, -8),
    ("lda T uses k", {"ta": "t", "k": 2, "lda": 2, "lda2": 8}, 0),
    ("ldb<k", {"ldb": 3}, -11),
    ("ldc<m", {"ldc": 3}, -15),
    ("lda2<0", {"lda2": -1}, -9),
    ("ldb2<0", {"ldb2": -16}, -12),
    ("ldc2<ldc*n", {"ldc2": 15}, -16),
    ("ldc2 unchecked at batch 1", {"ldc2": 0, "batch": 1}, 0),
    ("broadcast A (lda2=0)", {"lda2": 0}, 0),
    ("batch<0", {"batch": -1}, -17),
    ("m=0 quick", {"m": 0, "lda": 1}, 0),
]


@pytest.mark.parametrize("name,kw,want", VALIDATION, ids=[v[0] for v in VALIDATION])
def test_validation_codes(name, kw, want):
    a = _args(**kw)
    buf = np.zeros(4096)
    A = buf[:1000].copy()
    B = buf[:1000].copy()
    C = buf[:1000].copy()
    rc = oracle.gemm_batched(a["kind"], a["ta"], a["tb"], a["m"], a["n"], a["k"], a["alpha"], A,
                             a["lda"], a["lda2"], B, a["ldb"], a["ldb2"], a["beta"], C, a["ldc"],
                             a["ldc2"], a["batch"], alpha_ptr=a["alpha_ptr"],
                             beta_ptr=a["beta_ptr"])
    assert rc == want


def test_validation_null_and_alias():
    A = np.zeros(100)
    C = np.zeros(100)
    assert oracle.gemm_batched("d", "N", "N", 2, 2, 2, 1.0, None, 2, 4, A, 2, 4, 0.0, C, 2, 4, 2) == -7
    assert oracle.gemm_batched("d", "N", "N", 2, 2, 2, 1.0, A, 2, 4, None, 2, 4, 0.0, C, 2, 4, 2) == -10
    assert oracle.gemm_batched("d", "N", "N", 2, 2, 2, 1.0, A, 2, 4, A, 2, 4, 0.0, None, 2, 4, 2) == -14
    # alpha == 0: A/B may be NULL
    assert oracle.gemm_batched("d", "N", "N", 2, 2, 2, 0.0, None, 2, 4, None, 2, 4, 0.5, C, 2, 4, 2) == 0
    # C overlapping A -> -14; A and B may alias each other
    assert oracle.gemm_batched("d", "N", "N", 2, 2, 2, 1.0, A, 2, 4, A, 2, 4, 0.0, A, 2, 4, 2,
                               c_off=6) == -14
    # pointer variant positions
    assert oracle.gemm_batched_ptr("d", "N", "N", 2, 2, 2, 1.0, A, [0], 2, A, [0], 2, 0.0, C, [0],
                                   2, 1, beta_ptr=False) == -11
    assert oracle.gemm_batched_ptr("d", "N", "N", 2, 2, 2, 1.0, A, [0], 2, A, [0], 1, 0.0, C, [0],
                                   2, 1) == -10
    assert oracle.gemm_batched_ptr("d", "N", "N", 2, 2, 2, 1.0, A, [0], 2, A, [0], 2, 0.0, C, [0],
                                   1, 1) == -13
    assert oracle.gemm_batched_ptr("d", "N", "N", 2, 2, 2, 1.0, A, [0], 2, A, [0], 2, 0.0, C, [0],
                                   2, -1) == -14
    assert oracle.gemm_batched_ptr("d", "N", "N", 2, 2, 2, 1.0, A, [0], 2, A, [0], 2, 0.0, C, [0],
                                   2, 1, null_arrays=("B",)) == -9
    assert oracle.gemm_batched_ptr("d", "N", "N", 2, 2, 2, 1.0, A, [0], 2, A, [0], 2, 0.0, C, [0],
                                   2, 1, null_arrays=("C",)) == -12
