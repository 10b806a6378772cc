"""Parity of the tile-ring path: many tiles per CTA, every instance family.

At the parity sweep's batch sizes every CTA of the automatic grid gets one or two
tiles -- fewer than its pipeline stages -- so no stage is ever refilled and no
mbarrier phase flips.  Here the grid is capped (tx_set_max_ctas 1 and 7) so each
CTA loops over tens to hundreds of tiles: every stage is reused, both mbarrier
parities occur, TMA box coordinates of late tiles are exercised, and the ragged
last tile lands on an arbitrary stage.  Each result is compared with the oracle
element by element (Eq. (1); ops PAPER.md:240-243, 617-634;
epilogues PAPER.md:436-466) and bitwise with the automatic grid (results do not
depend on the grid, include/txgemm.h).
"""
from __future__ import annotations

import contextlib

import numpy as np
import pytest

import paper_1304_7053_b200 as tx
import txinputs
from gpu_util import check, run_lib, run_oracle, to_dev, torch_dtype
from helpers import OPS_CPLX, OPS_REAL, TOL, max_rel_err, random_case

pytestmark = pytest.mark.gpu

CAPS = (1, 7)
BATCH = 3001  # ragged: not a multiple of any tile size or of the 16-byte unit


def ops_for(kind):
    ops = OPS_CPLX if kind in "cz" else OPS_REAL
    return [(a, b) for a in ops for b in ops]


@contextlib.contextmanager
def max_ctas(v):
    prev = tx.set_max_ctas(v)
    try:
        yield
    finally:
        tx.set_max_ctas(prev)


def _ab(kind, tag, general=True):
    a = txinputs.scalar(kind, txinputs.stream_key(17, tag, "alpha"))
    return (a, txinputs.scalar(kind, txinputs.stream_key(17, tag, "beta"))) if general else (a, 0)


def _ring_case(kind, m, n, k, ta, tb, general, tag, batch=BATCH, pad=(0, 0), expect=None):
    A, B, C = random_case(kind, m, n, k, batch, ta, tb, seed=211, tag=tag, pad=pad)
    alpha, beta = _ab(kind, f"{tag}{kind}{m}{n}{k}{ta}{tb}", general)
    ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
    rc, auto, path = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
    assert rc == 0, tx.status_string(rc)
    if expect:
        assert path[0] in expect, path
    check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, auto, ref)
    for cap in CAPS:
        with max_ctas(cap):
            rc, got, path_c = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
        assert rc == 0, tx.status_string(rc)
        assert path_c == path, (cap, path_c, path)
        check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got, ref)
        assert np.array_equal(got.view(np.uint8), auto.view(np.uint8)), (kind, m, n, k, ta, tb, cap)


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("n", range(1, 17))
def test_ring_square_all_ops(kind, n):
    """Every AOT square instance (including the transpose-at-staging and swizzled
    tensor-copy instances the tables select) at >= S tiles per CTA."""
    for ta, tb in ops_for(kind):
        for general in (False, True):
            _ring_case(kind, n, n, n, ta, tb, general, "sq",
                       expect=("direct",) if n <= 2 else ("bulk", "bulk+tail"))


NONSQUARE = [(8, 16, 4), (16, 3, 16), (1, 16, 16), (5, 7, 3), (12, 7, 16), (16, 16, 8)]


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("mnk", NONSQUARE, ids=lambda t: "x".join(map(str, t)))
def test_ring_runtime_specialised_bulk(kind, mnk):
    """Runtime-specialised (NVRTC) bulk instances, swizzled TMA tiles included."""
    m, n, k = mnk
    for ta, tb in ops_for(kind):
        for general in (False, True):
            _ring_case(kind, m, n, k, ta, tb, general, "ns", expect=("bulk", "bulk+tail"))


@pytest.mark.parametrize("kind", "sdcz")
def test_ring_gather_padded(kind):
    for (m, n, k), (ta, tb) in (((16, 16, 16), ("T", "N")), ((5, 7, 3), ("N", "T")),
                                ((16, 3, 16), ("T", "T")), ((9, 9, 9), ("N", "N"))):
        if kind in "cz":
            ta, tb = ta.replace("T", "C"), tb
        for general in (False, True):
            _ring_case(kind, m, n, k, ta, tb, general, "gp", pad=(1, 3), expect=("gather",))


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("mnk", [(16, 16, 16), (24, 17, 32), (32, 32, 32)],
                         ids=lambda t: "x".join(map(str, t)))
def test_ring_sizes_beyond_16(kind, mnk):
    m, n, k = mnk
    for ta, tb in (("N", "N"), ("T", "C" if kind in "cz" else "T")):
        for general in (False, True):
            _ring_case(kind, m, n, k, ta, tb, general, "big", batch=1501)


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("which", ["A", "B", "AB"])
def test_ring_fixed_operand(kind, which):
    """ld2 = 0 (one matrix shared by every pair, the paper's §9 variant)."""
    import torch

    for n, (ta, tb) in ((16, ("N", "N")), (7, ("T", "N")), (12, ("N", "T"))):
        A, B, C = random_case(kind, n, n, n, BATCH, ta, tb, seed=212, tag="bc")
        if "A" in which:
            A.ld2 = 0
        if "B" in which:
            B.ld2 = 0
        alpha, beta = _ab(kind, f"bc{which}{n}")
        ref = run_oracle(kind, ta, tb, n, n, n, alpha, beta, A, B, C)
        outs = []
        for cap in (0,) + CAPS:
            with max_ctas(cap):
                rc, got, path = run_lib(kind, ta, tb, n, n, n, alpha, beta, A, B, C)
            assert rc == 0, tx.status_string(rc)
            check(kind, ta, tb, n, n, n, alpha, beta, A, B, C, got, ref)
            outs.append(got)
        for o in outs[1:]:
            assert np.array_equal(o.view(np.uint8), outs[0].view(np.uint8))


def _dev_scalar(kind, v):
    import torch

    return torch.tensor([v], dtype=torch_dtype(kind), device="cuda")


@pytest.mark.parametrize("kind", "sdcz")
def test_ring_device_scalars(kind):
    """Device-resident alpha/beta kernels (decided in-kernel) at many tiles per CTA,
    including run-time beta == 0 (C never read) and alpha == 0 (scale only)."""
    import torch

    ag, bg = _ab(kind, "devring")
    for (m, n, k), pad in (((16, 16, 16), (0, 0)), ((8, 16, 4), (0, 0)), ((5, 7, 3), (1, 2))):
        for alpha, beta in ((ag, bg), (ag, 0), (0, bg)):
            A, B, C = random_case(kind, m, n, k, BATCH, "T", "N", seed=213, tag="devring", pad=pad)
            if beta == 0:
                C.buf[C.mask()] = np.nan
            if alpha == 0:
                A.buf[:] = np.nan
                B.buf[:] = np.nan
            ref = run_oracle(kind, "T", "N", m, n, k, alpha, beta, A, B, C)
            outs = []
            for cap in (0,) + CAPS:
                dA, _ = to_dev(A)
                dB, _ = to_dev(B)
                dC, _ = to_dev(C)
                with max_ctas(cap):
                    rc = tx.tx_gemm_batched_dev(kind, "T", "N", m, n, k, _dev_scalar(kind, alpha),
                                                dA, A.ld, A.ld2, dB, B.ld, B.ld2,
                                                _dev_scalar(kind, beta), dC, C.ld, C.ld2, C.batch)
                assert rc == 0, tx.status_string(rc)
                torch.cuda.synchronize()
                got = dC.cpu().numpy()
                if alpha == 0:  # C <- beta*C; den = |beta||C0| (A, B are NaN, never read)
                    den = abs(beta) * np.abs(C.dense().astype(np.complex128))
                    assert max_rel_err(kind, C.dense(got), C.dense(ref), den) <= TOL[kind]
                else:
                    check(kind, "T", "N", m, n, k, alpha, beta, A, B, C, got, ref)
                outs.append(got)
            for o in outs[1:]:
                assert np.array_equal(o.view(np.uint8), outs[0].view(np.uint8))


def _ptr_run(kind, m, n, k, ta, tb, alpha, beta, A, B, C, perm, byte_off=0):
    """Pointer-array call over device copies, matrix p at its strided place, pointers
    permuted; byte_off shifts every matrix (the buffers are re-based by that many bytes)."""
    import torch

    outs = []
    for cap in (0,) + CAPS:
        dA, _ = to_dev(A)
        dB, _ = to_dev(B)
        dC, _ = to_dev(C)
        es = dA.element_size()
        if byte_off:  # place the same values at an offset of byte_off bytes
            sh = byte_off // es
            dA2 = torch.zeros(dA.numel() + sh + 1, dtype=dA.dtype, device="cuda")
            dB2 = torch.zeros(dB.numel() + sh + 1, dtype=dB.dtype, device="cuda")
            dC2 = torch.zeros(dC.numel() + sh + 1, dtype=dC.dtype, device="cuda")
            dA2[sh:sh + dA.numel()] = dA
            dB2[sh:sh + dB.numel()] = dB
            dC2[sh:sh + dC.numel()] = dC
            bases = [x.data_ptr() + sh * es for x in (dA2, dB2, dC2)]
        else:
            bases = [x.data_ptr() for x in (dA, dB, dC)]
        pa = torch.tensor(A.offsets()[perm] * es + bases[0], device="cuda")
        pb = torch.tensor(B.offsets()[perm] * es + bases[1], device="cuda")
        pc = torch.tensor(C.offsets()[perm] * es + bases[2], device="cuda")
        with max_ctas(cap):
            rc = tx.tx_gemm_batched_ptr(kind, ta, tb, m, n, k, alpha, pa, A.ld, pb, B.ld, beta, pc,
                                        C.ld, C.batch)
        assert rc == 0, tx.status_string(rc)
        assert tx.last_path()[0] == "ptr"
        torch.cuda.synchronize()
        if byte_off:
            got = dC2[sh:sh + dC.numel()].cpu().numpy()
        else:
            got = dC.cpu().numpy()
        outs.append(got)
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint8), outs[0].view(np.uint8))
    return outs[0]


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("mnk", [(5, 7, 3), (4, 6, 16), (8, 16, 4), (16, 16, 16), (16, 3, 16)],
                         ids=lambda t: "x".join(map(str, t)))
def test_ring_pointer_arrays(kind, mnk):
    """Pointer arrays (element gather, 16-byte chunk gather, per-matrix bulk copies --
    chosen by matrix size) with permuted pointers at many tiles per CTA."""
    m, n, k = mnk
    for ta, tb in (("N", "N"), ("T", "C" if kind in "cz" else "T")):
        for general in (False, True):
            A, B, C = random_case(kind, m, n, k, BATCH, ta, tb, seed=214, tag="ptrring")
            alpha, beta = _ab(kind, f"pr{m}{n}{k}{ta}{tb}", general)
            perm = np.random.default_rng(m * 100 + n).permutation(BATCH)
            got = _ptr_run(kind, m, n, k, ta, tb, alpha, beta, A, B, C, perm)
            ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
            check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got, ref)


@pytest.mark.parametrize("kind", "sdcz")
def test_pointer_arrays_not_16_byte_aligned(kind):
    """Pointers aligned to the element size but not to 16 bytes: the per-matrix bulk
    kernel (packed matrices >= 512 B) copies those matrices synchronously before the
    stage's barrier arrives (the whole tile may be unaligned).  s: +4 B, +8 B, +12 B;
    d, c: +8 B; z is always 16-byte aligned."""
    es = {"s": 4, "d": 8, "c": 8, "z": 16}[kind]
    offs = [o for o in (4, 8, 12) if o % es == 0 and o % 16 != 0]
    if not offs:
        pytest.skip("element size 16: every aligned element pointer is 16-byte aligned")
    # pad ld2 by one element: consecutive matrices alternate between aligned and not,
    # so tiles mix bulk-copied and synchronously copied matrices
    for n, pad, off in [(16, (0, 0), o) for o in offs] + [(12, (0, 0), offs[0]), (16, (0, 1), 0),
                                                       (12, (0, 1), offs[0])]:
        for general in (False, True):
                A, B, C = random_case(kind, n, n, n, BATCH, "N", "T", seed=215, tag="unal", pad=pad)
                alpha, beta = _ab(kind, f"unal{n}{off}", general)
                perm = np.random.default_rng(off).permutation(BATCH)
                got = _ptr_run(kind, n, n, n, "N", "T", alpha, beta, A, B, C, perm, byte_off=off)
                ref = run_oracle(kind, "N", "T", n, n, n, alpha, beta, A, B, C)
                check(kind, "N", "T", n, n, n, alpha, beta, A, B, C, got, ref)
