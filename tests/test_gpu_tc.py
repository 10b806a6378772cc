"""Parity of the tensor-core (tcgen05 split-TF32) kernel for s / c against the oracle.

The kernel (csrc/tx_tc.cuh) serves packed single-precision batches
beyond 16 ("can be easily extended to larger sizes").  tx_set_tc(1)
forces it wherever it applies so small shapes are covered too; every case checks the
path and compares with the oracle element by element (north-star tolerance 1e-5,
normalised by |alpha| sum |op(A)||op(B)| + |beta||C0|), or bitwise on integer inputs.
"""
from __future__ import annotations

import contextlib

import numpy as np
import pytest

import paper_1304_7053_b200 as tx
import txinputs
from gpu_util import check, run_lib, run_oracle
from helpers import OPS_CPLX, OPS_REAL, random_case

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def tc_forced(mode=1, max_ctas=0):
    from paper_1304_7053_b200 import binding

    prev = binding.set_tc(mode)
    prev_ctas = binding.lib().tx_set_max_ctas(max_ctas)
    try:
        yield
    finally:
        binding.set_tc(prev)
        binding.lib().tx_set_max_ctas(prev_ctas)


def ops_for(kind):
    ops = OPS_CPLX if kind == "c" else OPS_REAL
    return [(a, b) for a in ops for b in ops]


def _ab(kind, tag, general):
    a = txinputs.scalar(kind, txinputs.stream_key(17, tag, "alpha"))
    return (a, txinputs.scalar(kind, txinputs.stream_key(17, tag, "beta"))) if general else (a, 0)


def _run(kind, m, n, k, batch, ta, tb, general, tag, dist="uniform"):
    A, B, C = random_case(kind, m, n, k, batch, ta, tb, seed=31, tag=tag, dist=dist)
    alpha, beta = _ab(kind, f"{tag}{m}{n}{k}{ta}{tb}", general)
    if dist == "int":
        alpha = txinputs.scalar(kind, 3, dist="int")
        beta = txinputs.scalar(kind, 4, dist="int") if general else 0
    rc, got, path = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
    assert rc == 0, tx.status_string(rc)
    assert path[0] in ("tc", "tc+tail"), path
    ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
    return A, B, C, alpha, beta, got, ref


SHAPES_S = [(64, 64, 64), (33, 33, 33), (48, 48, 48), (40, 24, 56), (17, 64, 5), (64, 1, 64),
            (1, 64, 33), (16, 16, 16), (8, 8, 8), (3, 5, 7), (64, 17, 40), (20, 31, 9)]
SHAPES_C = [(32, 32, 32), (17, 17, 17), (24, 24, 24), (20, 31, 9), (32, 5, 32), (1, 32, 32),
            (32, 32, 1), (16, 16, 16), (5, 6, 7), (31, 29, 27)]


@pytest.mark.parametrize("kind,mnk", [("s", t) for t in SHAPES_S] + [("c", t) for t in SHAPES_C],
                         ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
def test_tc_matches_oracle(kind, mnk):
    """Every op pair x {beta == 0, general}, 301 pairs (several tiles, ragged tail)."""
    m, n, k = mnk
    with tc_forced():
        for ta, tb in ops_for(kind):
            for general in (False, True):
                A, B, C, alpha, beta, got, ref = _run(kind, m, n, k, 301, ta, tb, general, "tc")
                check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got, ref)


@pytest.mark.parametrize("kind,mnk", [("s", (64, 64, 64)), ("s", (37, 41, 43)), ("s", (24, 24, 24)),
                                      ("c", (32, 32, 32)), ("c", (19, 23, 29)), ("c", (8, 8, 8))],
                         ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
def test_tc_integer_inputs_bit_exact(kind, mnk):
    """Integer entries in [-4, 4]: the hi parts are exact, the lo parts zero, every sum
    exact -- the tensor-core result equals the oracle bitwise."""
    m, n, k = mnk
    with tc_forced():
        for ta, tb in ops_for(kind):
            for general in (False, True):
                _, _, _, _, _, got, ref = _run(kind, m, n, k, 203, ta, tb, general, "tcint", "int")
                assert np.array_equal(got, ref), (kind, mnk, ta, tb, general)


@pytest.mark.parametrize("kind,mnk", [("s", (64, 64, 64)), ("s", (33, 20, 47)), ("c", (32, 32, 32)),
                                      ("c", (21, 17, 30))],
                         ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
@pytest.mark.parametrize("ctas", [1, 7])
def test_tc_ring_reuse(kind, mnk, ctas):
    """Grid capped so each CTA loops over many tiles: every stage refilled, both
    operand buffers and both TMEM accumulators reused, mbarrier parities flipping."""
    m, n, k = mnk
    ta, tb = ("T", "N") if kind == "s" else ("C", "T")
    with tc_forced(max_ctas=ctas):
        for general in (False, True):
            A, B, C, alpha, beta, got, ref = _run(kind, m, n, k, 613, ta, tb, general, "tcring")
            check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got, ref)
    # the automatic grid gives the same bits (each pair's arithmetic is independent of the grid)
    with tc_forced():
        _, _, _, _, _, got2, _ = _run(kind, m, n, k, 613, ta, tb, True, "tcring")
    assert np.array_equal(got2, got)


@pytest.mark.parametrize("kind", "sc")
def test_tc_beta0_never_reads_C(kind):
    m = n = k = 32 if kind == "c" else 48
    A, B, C = random_case(kind, m, n, k, 257, seed=6, tag="tcnan", c_sentinel=np.nan)
    C.buf[:] = np.nan
    alpha = txinputs.scalar(kind, 9)
    with tc_forced():
        rc, got, path = run_lib(kind, "N", "N", m, n, k, alpha, 0, A, B, C)
    assert rc == 0 and path[0] in ("tc", "tc+tail")
    assert np.all(np.isfinite(C.dense(got)))
    ref = run_oracle(kind, "N", "N", m, n, k, alpha, 0, A, B, C)
    check(kind, "N", "N", m, n, k, alpha, 0, A, B, C, got, ref)


@pytest.mark.parametrize("kind,n", [("s", 64), ("s", 45), ("c", 32), ("c", 29)])
def test_tc_default_rule_and_batch_edges(kind, n):
    """The automatic rule picks the tensor-core kernel at these sizes; batches 1, 2, 3,
    149 (one pair per SM and a few over), and a large odd batch."""
    for batch in (1, 2, 3, 149, 1001):
        A, B, C = random_case(kind, n, n, n, batch, "N", "N", seed=8, tag="tcedge")
        alpha, beta = _ab(kind, f"edge{n}{batch}", True)
        rc, got, path = run_lib(kind, "N", "N", n, n, n, alpha, beta, A, B, C)
        assert rc == 0 and path[0] in ("tc", "tc+tail"), path
        ref = run_oracle(kind, "N", "N", n, n, n, alpha, beta, A, B, C)
        check(kind, "N", "N", n, n, n, alpha, beta, A, B, C, got, ref)


@pytest.mark.parametrize("kind,mnk", [("s", (51, 51, 51)), ("s", (63, 61, 59)), ("c", (31, 29, 27)),
                                      ("c", (17, 19, 23))],
                         ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
@pytest.mark.parametrize("misalign", [0, 1, 3])
def test_tc_any_element_alignment(kind, mnk, misalign):
    """Packed batches whose per-pair byte sizes are not multiples of 16 and whose bases are
    only element-aligned: the kernel copies the 16-byte-aligned windows covering each
    tile, so every pair -- and the whole batch, no tail launch -- runs on it."""
    m, n, k = mnk
    with tc_forced():
        for general in (False, True):
            A, B, C = random_case(kind, m, n, k, 157, "N", "T", seed=41, tag="tcwin")
            alpha, beta = _ab(kind, f"win{m}{misalign}", general)
            rc, got, path = run_lib(kind, "N", "T", m, n, k, alpha, beta, A, B, C, misalign=misalign)
            assert rc == 0 and path == ("tc", 1), path
            ref = run_oracle(kind, "N", "T", m, n, k, alpha, beta, A, B, C)
            check(kind, "N", "T", m, n, k, alpha, beta, A, B, C, got, ref)
