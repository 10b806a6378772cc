"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

Element by element on the same seeded inputs: within 1e-5 (s, c) / 1e-13 (d, z)
normalised by |alpha| sum|op(A)||op(B)| + |beta||C0| (BASELINE.json north_star),
and bit-exact where the inputs make every order of summation exact.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1304_7053_b200 as tx
import txinputs
from gpu_util import check, run_lib, run_oracle, to_dev, torch_dtype
from helpers import (NP, OPS_CPLX, OPS_REAL, TOL, Operand, dense_at, denominators,
                     denominators_dense, max_rel_err, random_case, stored_shape)

pytestmark = pytest.mark.gpu


def ops_for(kind):
    ops = OPS_CPLX if kind in "cz" else OPS_REAL
    return [(a, b) for a in ops for b in ops]


def _ab(kind, tag, general=True):
    if not general:
        return txinputs.scalar(kind, txinputs.stream_key(7, tag, "alpha")), 0
    return (txinputs.scalar(kind, txinputs.stream_key(7, tag, "alpha")),
            txinputs.scalar(kind, txinputs.stream_key(7, tag, "beta")))


def _case(kind, m, n, k, batch, ta, tb, general, tag, **kw):
    A, B, C = random_case(kind, m, n, k, batch, ta, tb, seed=101, tag=tag, **kw)
    alpha, beta = _ab(kind, f"{tag}{kind}{m}{n}{k}{ta}{tb}", general)
    rc, got, path = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
    assert rc == 0, tx.status_string(rc)
    ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
    err = check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got, ref)
    return err, path, (A, B, C, alpha, beta, got, ref)


# ------------------------------------------------------------ the full sweep
@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("n", range(1, 17))
def test_square_sweep_all_ops(kind, n):
    """Config 3 shape at reduced batch: every op pair, beta == 0 and general,
    1003 pairs (several tiles and a ragged tail)."""
    for ta, tb in ops_for(kind):
        for general in (False, True):
            err, path, _ = _case(kind, n, n, n, 1003, ta, tb, general, "sweep")
            assert path[0] in (("direct",) if n <= 2 else ("bulk", "bulk+tail")), path


NONSQUARE = [(8, 16, 4), (16, 3, 16), (1, 16, 16), (16, 16, 1), (5, 7, 3), (16, 1, 7), (2, 9, 13),
             (5, 6, 16), (12, 7, 16)]


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("mnk", NONSQUARE, ids=lambda t: "x".join(map(str, t)))
def test_nonsquare(kind, mnk):
    m, n, k = mnk
    for ta, tb in ops_for(kind):
        for general in (False, True):
            _case(kind, m, n, k, 517, ta, tb, general, "ns")


# ---------------------------------------------------------- exactness / edge
@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("n", [1, 3, 4, 8, 13, 16])
def test_integer_inputs_bit_exact(kind, n):
    """Integer entries in [-4, 4], integer alpha/beta: every summation order is
    exact, so GPU == oracle bitwise (compared with ==, +-0 allowed)."""
    for ta, tb in ops_for(kind):
        A, B, C = random_case(kind, n, n, n, 777, ta, tb, seed=5, tag="int", dist="int")
        alpha = txinputs.scalar(kind, 3, dist="int")
        beta = txinputs.scalar(kind, 4, dist="int")
        rc, got, _ = run_lib(kind, ta, tb, n, n, n, alpha, beta, A, B, C)
        assert rc == 0
        ref = run_oracle(kind, ta, tb, n, n, n, alpha, beta, A, B, C)
        assert np.array_equal(got, ref), (kind, n, ta, tb)


@pytest.mark.parametrize("kind", "sdcz")
def test_beta0_never_reads_C(kind):
    for n in (2, 7, 16):
        A, B, C = random_case(kind, n, n, n, 600, seed=6, tag="nanC", c_sentinel=np.nan)
        C.buf[:] = np.nan
        alpha = txinputs.scalar(kind, 9)
        rc, got, _ = run_lib(kind, "N", "N", n, n, n, alpha, 0, A, B, C)
        assert rc == 0
        assert np.all(np.isfinite(C.dense(got)))
        ref = run_oracle(kind, "N", "N", n, n, n, alpha, 0, A, B, C)
        check(kind, "N", "N", n, n, n, alpha, 0, A, B, C, got, ref)


@pytest.mark.parametrize("kind", "sdcz")
def test_alpha0_and_k0_scale_C(kind):
    for alpha, k in ((0, 5), (1.5, 0)):
        A, B, C = random_case(kind, 5, 6, max(k, 1), 300, seed=7, tag="a0", dist="int")
        A.buf[:] = np.nan
        B.buf[:] = np.nan
        beta = txinputs.scalar(kind, 5, dist="int")
        rc, got, path = run_lib(kind, "N", "N", 5, 6, k, alpha, beta, A, B, C)
        assert rc == 0 and path[0] == "scale"
        ref = run_oracle(kind, "N", "N", 5, 6, k, alpha, beta, A, B, C)
        assert np.array_equal(got, ref)
        # beta == 0: C <- 0 without reading C
        C.buf[:] = np.nan
        rc, got, _ = run_lib(kind, "N", "N", 5, 6, k, alpha, 0, A, B, C)
        assert rc == 0 and np.all(C.dense(got) == 0)


@pytest.mark.parametrize("kind", "sdcz")
def test_padded_layout_and_sentinels(kind):
    """General strided path (ld > rows, ld2 > ld*cols): same values as the oracle,
    pad entries of C bitwise untouched."""
    for n, ta, tb in ((5, "N", "T"), (16, "T", "N"), (9, "C", "C")):
        if kind in "sd":
            ta, tb = ta.replace("C", "T"), tb.replace("C", "T")
        A, B, C = random_case(kind, n, n, n, 333, ta, tb, seed=8, tag="pad", pad=(3, 5),
                              c_sentinel=-3.75)
        alpha, beta = _ab(kind, "pad")
        rc, got, path = run_lib(kind, ta, tb, n, n, n, alpha, beta, A, B, C)
        assert rc == 0 and path[0] == "gather", path
        ref = run_oracle(kind, ta, tb, n, n, n, alpha, beta, A, B, C)
        check(kind, ta, tb, n, n, n, alpha, beta, A, B, C, got, ref)
        mask = C.mask()
        assert np.array_equal(got[~mask].view(np.uint8), C.buf[~mask].view(np.uint8))


@pytest.mark.parametrize("kind", "sdcz")
def test_misaligned_base_uses_gather(kind):
    A, B, C = random_case(kind, 8, 8, 8, 257, seed=9, tag="mis")
    alpha, beta = _ab(kind, "mis")
    rc, got, path = run_lib(kind, "N", "N", 8, 8, 8, alpha, beta, A, B, C, misalign=1)
    assert rc == 0
    if kind != "z":
        assert path[0] == "gather"
    ref = run_oracle(kind, "N", "N", 8, 8, 8, alpha, beta, A, B, C)
    check(kind, "N", "N", 8, 8, 8, alpha, beta, A, B, C, got, ref)


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("which", ["A", "B", "AB"])
def test_fixed_operand_ld2_zero(kind, which):
    """lda2 = 0 / ldb2 = 0: one A (or B) for every pair -- the paper's fixed-operand
    variant (§9).  Packed otherwise, it runs the bulk kernel with the
    shared operand resident in shared memory (runtime-specialised instance)."""
    from paper_1304_7053_b200 import binding

    for (m, n, k), ta, tb, batch in (((6, 6, 6), "N", "N", 411), ((16, 16, 16), "T", "N", 1000),
                                     ((8, 16, 4), "N", "T", 777), ((5, 3, 7), "T", "T", 513)):
        if kind in "cz":
            ta = ta.replace("T", "C")
        A, B, C = random_case(kind, m, n, k, batch, ta, tb, seed=10, tag="bc" + which)
        ra, ca = stored_shape(ta, m, k)
        rb, cb = stored_shape(tb, k, n)
        if "A" in which:
            A = Operand(kind, ra, ca, 1, txinputs.stream_key(10, "bcA", m, n, k))
            A.ld2, A.batch = 0, batch
        if "B" in which:
            B = Operand(kind, rb, cb, 1, txinputs.stream_key(10, "bcB", m, n, k))
            B.ld2, B.batch = 0, batch
        for general in (False, True):
            alpha, beta = _ab(kind, "bc" + which, general)
            rc, got, path = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
            assert rc == 0
            if binding.jit_compiled() >= 0:
                assert path[0] in ("bulk", "bulk+tail"), path
            ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
            check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got, ref)


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("batch", [1, 2, 3, 15, 17, 4099])
def test_batch_edges(kind, batch):
    for n in (1, 3, 16):
        _case(kind, n, n, n, batch, "N", "N", True, f"be{batch}")


# ---------------------------------------- A tile by TMA tensor copy (ASW)
@pytest.mark.parametrize("kind", "dcz")
@pytest.mark.parametrize("batch", [1, 5, 16, 17, 100, 1003])
def test_transposed_a_tensor_copy_tiles(kind, batch):
    """n = 16 with op(A) = T/C on 8/16-byte types: the bulk instances may load A with
    a swizzled TMA tensor copy whose last box runs past the batch (zero-filled).
    Ragged batches against the oracle, and bitwise against the pointer-array path
    (a different data mover, same summation order)."""
    import torch

    for ta in ("T", "C") if kind in "cz" else ("T",):
        for tb in ("N", "T"):
            for general in (False, True):
                err, path, (A, B, C, alpha, beta, got, ref) = _case(
                    kind, 16, 16, 16, batch, ta, tb, general, f"asw{batch}")
                assert path[0] in ("bulk", "bulk+tail"), path
                dA, _ = to_dev(A)
                dB, _ = to_dev(B)
                dC, _ = to_dev(C)
                es = dA.element_size()
                pa = torch.tensor(A.offsets() * es + dA.data_ptr(), device="cuda")
                pb = torch.tensor(B.offsets() * es + dB.data_ptr(), device="cuda")
                pc = torch.tensor(C.offsets() * es + dC.data_ptr(), device="cuda")
                rc = tx.tx_gemm_batched_ptr(kind, ta, tb, 16, 16, 16, alpha, pa, A.ld, pb, B.ld,
                                            beta, pc, C.ld, C.batch)
                assert rc == 0
                got_ptr = dC.cpu().numpy()
                assert np.array_equal(got_ptr.view(np.uint8), got.view(np.uint8))


@pytest.mark.parametrize("kind", "dcz")
def test_swizzled_gather_layouts(kind):
    """Gather instances may place op(A) = T/C and op(B) = N copies in the 128-byte-
    swizzled layout (k * sizeof(T) a multiple of 128 B; m, n not multiples of 8 check
    the per-matrix line offset): pointer arrays (16-byte chunks, permuted) and a padded strided layout
    (element copies) against the oracle; pointer arrays bitwise against the packed
    strided call."""
    import torch

    shapes = [(16, 3, 16), (5, 3, 16), (12, 7, 16), (1, 16, 16), (4, 6, 16)] + \
        ([(3, 4, 8)] if kind == "z" else [])
    for (m, n, k) in shapes:
        for ta in ("N", "T", "C") if kind in "cz" else ("N", "T"):
            for tb in ("N", "T"):
                alpha, beta = _ab(kind, f"swg{m}{n}{k}")
                A, B, C = random_case(kind, m, n, k, 517, ta, tb, seed=5, tag="swg")
                dA, _ = to_dev(A)
                dB, _ = to_dev(B)
                dC, _ = to_dev(C)
                es = dA.element_size()
                perm = np.random.default_rng(4).permutation(C.batch)
                pa = torch.tensor(A.offsets()[perm] * es + dA.data_ptr(), device="cuda")
                pb = torch.tensor(B.offsets()[perm] * es + dB.data_ptr(), device="cuda")
                pc = torch.tensor(C.offsets()[perm] * es + dC.data_ptr(), device="cuda")
                rc = tx.tx_gemm_batched_ptr(kind, ta, tb, m, n, k, alpha, pa, A.ld, pb, B.ld,
                                            beta, pc, C.ld, C.batch)
                assert rc == 0
                got_ptr = dC.cpu().numpy()
                ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
                check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got_ptr, ref)
                # the packed strided call (bulk kernel, plain layout): same sums, same bits
                rc, got_str, _ = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
                assert rc == 0
                assert np.array_equal(got_str.view(np.uint8), got_ptr.view(np.uint8))
                Ap, Bp, Cp = random_case(kind, m, n, k, 517, ta, tb, seed=5, tag="swg", pad=(2, 3))
                rc, got_pad, path = run_lib(kind, ta, tb, m, n, k, alpha, beta, Ap, Bp, Cp)
                assert rc == 0 and path[0] == "gather", path
                refp = run_oracle(kind, ta, tb, m, n, k, alpha, beta, Ap, Bp, Cp)
                check(kind, ta, tb, m, n, k, alpha, beta, Ap, Bp, Cp, got_pad, refp)


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("batch", [1, 37, 1003])
def test_pointer_arrays_odd_sizes_any_alignment(kind, batch):
    """Packed matrices whose byte sizes are not multiples of 16, at arbitrary element
    offsets (so every 16-byte alignment occurs): the covering-chunk gather (U16) reads
    partial first / last chunks element by element.  Against the oracle's pointer
    variant on the same offsets; C entries outside the matrices stay untouched."""
    import torch

    rng = np.random.default_rng(batch)
    for (m, n, k) in ((5, 7, 3), (3, 3, 3), (1, 1, 1), (7, 2, 5)):
        for ta, tb in (("N", "N"), ("T", "C" if kind in "cz" else "T")):
            for general in (False, True):
                ra, ca = (m, k) if ta == "N" else (k, m)
                rb, cb = (k, n) if tb == "N" else (n, k)
                sa, sb, sc = ra * ca, rb * cb, m * n
                # each matrix at a random element offset: gaps of 0..7 elements
                def offs(size):
                    gaps = rng.integers(0, 8, batch)
                    return np.cumsum(gaps + size) - size
                oa, ob, oc = offs(sa), offs(sb), offs(sc)
                key = lambda nm: txinputs.stream_key(9, "u16", kind, m, n, k, ta, tb, batch, nm)
                hA = txinputs.values_numpy(kind, key("A"), 0, int(oa[-1]) + sa + 8)
                hB = txinputs.values_numpy(kind, key("B"), 0, int(ob[-1]) + sb + 8)
                hC = txinputs.values_numpy(kind, key("C"), 0, int(oc[-1]) + sc + 8)
                alpha, beta = _ab(kind, f"u16{m}{n}{k}", general)
                dA, dB, dC = (torch.from_numpy(x.copy()).cuda() for x in (hA, hB, hC))
                es = dA.element_size()
                pa = torch.tensor(oa * es + dA.data_ptr(), device="cuda")
                pb = torch.tensor(ob * es + dB.data_ptr(), device="cuda")
                pc = torch.tensor(oc * es + dC.data_ptr(), device="cuda")
                rc = tx.tx_gemm_batched_ptr(kind, ta, tb, m, n, k, alpha, pa, ra, pb, rb, beta, pc,
                                            m, batch)
                assert rc == 0
                got = dC.cpu().numpy()
                ref = hC.copy()
                assert oracle.gemm_batched_ptr(kind, ta, tb, m, n, k, alpha, hA, oa, ra, hB, ob, rb,
                                               beta, ref, oc, m, batch) == 0
                mask = np.zeros(len(hC), bool)
                for o in oc:
                    mask[o:o + sc] = True
                assert np.array_equal(got[~mask].view(np.uint8), hC[~mask].view(np.uint8))
                den = denominators_dense(kind, ta, tb, alpha, beta, dense_at(hA, oa, ra, ca, ra),
                                         dense_at(hB, ob, rb, cb, rb), dense_at(hC, oc, m, n, m))
                err = max_rel_err(kind, dense_at(got, oc, m, n, m), dense_at(ref, oc, m, n, m), den)
                assert err <= TOL[kind], (m, n, k, ta, tb, err)


# ------------------------------------------------------ pointer-array layout
@pytest.mark.parametrize("kind", "sdcz")
def test_pointer_array_equals_strided_and_oracle(kind):
    import torch

    for (m, n, k) in ((8, 16, 4), (16, 3, 16), (7, 7, 7)):
        for ta, tb in ops_for(kind)[::2]:
            A, B, C = random_case(kind, m, n, k, 999, ta, tb, seed=11, tag="ptr")
            alpha, beta = _ab(kind, "ptr")
            rc, got_strided, _ = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
            assert rc == 0
            perm = np.random.default_rng(2).permutation(C.batch)
            dA, _ = to_dev(A)
            dB, _ = to_dev(B)
            dC, _ = to_dev(C)
            es = dA.element_size()
            pa = torch.tensor(A.offsets()[perm] * es + dA.data_ptr(), device="cuda")
            pb = torch.tensor(B.offsets()[perm] * es + dB.data_ptr(), device="cuda")
            pc = torch.tensor(C.offsets()[perm] * es + dC.data_ptr(), device="cuda")
            rc = tx.tx_gemm_batched_ptr(kind, ta, tb, m, n, k, alpha, pa, A.ld, pb, B.ld, beta, pc,
                                        C.ld, C.batch)
            assert rc == 0 and tx.last_path()[0] == "ptr"
            got = dC.cpu().numpy()
            # each pair is independent: permuting the pointers permutes nothing in the result
            assert np.array_equal(got.view(np.uint8), got_strided.view(np.uint8))
            ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
            check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got, ref)


# ------------------------------------------------------------- determinism
@pytest.mark.parametrize("kind", "sz")
def test_deterministic_across_grid_sizes(kind):
    n = 16
    A, B, C = random_case(kind, n, n, n, 5000, seed=12, tag="det")
    alpha, beta = _ab(kind, "det")
    outs = []
    for cap in (0, 1, 7, 148):
        prev = tx.set_max_ctas(cap)
        try:
            rc, got, _ = run_lib(kind, "N", "T", n, n, n, alpha, beta, A, B, C)
        finally:
            tx.set_max_ctas(prev)
        assert rc == 0
        outs.append(got)
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint8), outs[0].view(np.uint8))


# ----------------------------------------------------------- host-buffer API
@pytest.mark.parametrize("kind", "sdcz")
def test_hostio_equals_device_path(kind):
    import torch

    n, batch = 10, 2000
    A, B, C = random_case(kind, n, n, n, batch, seed=13, tag="hio")
    alpha, beta = _ab(kind, "hio")
    rc, got_dev, _ = run_lib(kind, "N", "N", n, n, n, alpha, beta, A, B, C)
    hA = torch.from_numpy(A.buf.copy()).pin_memory()
    hB = torch.from_numpy(B.buf.copy()).pin_memory()
    hC = torch.from_numpy(C.buf.copy()).pin_memory()
    dA, dB, dC = (torch.empty_like(x, device="cuda") for x in (hA, hB, hC))
    rc = tx.tx_gemm_batched_hostio(kind, "N", "N", n, n, n, alpha, hA.data_ptr(), A.ld, A.ld2,
                                   hB.data_ptr(), B.ld, B.ld2, beta, hC.data_ptr(), C.ld, C.ld2,
                                   batch, torch.cuda.current_stream(), dA, dB, dC)
    assert rc == 0
    torch.cuda.synchronize()
    assert np.array_equal(hC.numpy().view(np.uint8), got_dev.view(np.uint8))


# ------------------------------------------------- tensor API
def test_tensor_api_matches_torch_layout():
    import torch

    kind, m, n, k, batch = "d", 5, 6, 7, 300
    A, B, C = random_case(kind, m, n, k, batch, seed=14, tag="tapi")
    At = torch.from_numpy(A.buf.copy()).cuda().view(batch, k, m).transpose(1, 2)
    Bt = torch.from_numpy(B.buf.copy()).cuda().view(batch, n, k).transpose(1, 2)
    Ct = torch.from_numpy(C.buf.copy()).cuda().view(batch, n, m).transpose(1, 2)
    tx.gemm_batched(At, Bt, Ct, "N", "N", 0.5, 0.25)
    torch.cuda.synchronize()
    ref = run_oracle(kind, "N", "N", m, n, k, 0.5, 0.25, A, B, C)
    got = Ct.transpose(1, 2).contiguous().view(-1).cpu().numpy()
    check(kind, "N", "N", m, n, k, 0.5, 0.25, A, B, C, got, ref)


# ---------------------------------------------- runtime specialisation (NVRTC)
@pytest.mark.parametrize("kind", "sdcz")
def test_jit_instances_match_aot_generic_bitwise(kind):
    """Non-square packed (bulk), padded (gather) and pointer-array calls run
    runtime-specialised sm_100a instances; with JIT disabled the generic-size AOT
    kernels run instead.  Both accumulate in ascending l: results are bitwise equal,
    and both match the oracle."""
    import torch
    from paper_1304_7053_b200 import binding

    if binding.jit_compiled() < 0:
        pytest.skip("NVRTC unavailable")
    cases = [((8, 16, 4), (0, 0), "N", "T"), ((5, 7, 3), (2, 3), "T", "N"),
             ((16, 3, 16), (0, 0), "T", "T")]
    for (m, n, k), pad, ta, tb in cases:
        if kind in "cz":
            tb = tb.replace("T", "C")
        A, B, C = random_case(kind, m, n, k, 613, ta, tb, seed=31, tag="jit", pad=pad)
        alpha, beta = _ab(kind, "jit")
        outs = []
        for jit in (True, False):
            prev = binding.set_jit(jit)
            try:
                rc, got, path = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
                used_jit = binding.last_path_jit()
            finally:
                binding.set_jit(prev)
            assert rc == 0 and used_jit == jit, (path, used_jit)
            outs.append(got)
        assert np.array_equal(outs[0].view(np.uint8), outs[1].view(np.uint8))
        ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
        check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, outs[0], ref)


# ------------------------------------------------- device-resident alpha / beta
def _dev_scalar(kind, v):
    import torch

    return torch.tensor([v], dtype=torch_dtype(kind), device="cuda")


@pytest.mark.parametrize("kind", "sdcz")
def test_device_alpha_beta(kind):
    """tx_gemm_batched_dev_* read alpha/beta on the device and decide
    beta == 0 / alpha == 0 in-kernel: same results as the host-scalar call and the oracle;
    beta == 0 never reads C (NaN-filled), alpha == 0 never reads A, B (NaN-filled)."""
    import torch

    ab_gen = _ab(kind, "dev")
    cases = [ab_gen, (ab_gen[0], 0), (0, ab_gen[1]), (0, 0), (0, 1), (1, 1)]
    for (m, n, k), pad in (((16, 16, 16), (0, 0)), ((8, 16, 4), (0, 0)), ((5, 7, 3), (1, 2)),
                           ((6, 6, 0), (0, 0))):
        for alpha, beta in cases:
            A, B, C = random_case(kind, m, n, max(k, 1), 613, "N", "T", seed=41, tag="dev", pad=pad)
            if alpha == 0 or k == 0:
                A.buf[:] = np.nan
                B.buf[:] = np.nan
            if beta == 0:
                C.buf[C.mask()] = np.nan
            dA, _ = to_dev(A)
            dB, _ = to_dev(B)
            dC, _ = to_dev(C)
            es = dA.element_size()
            rc = tx.tx_gemm_batched_dev(kind, "N", "T", m, n, k, _dev_scalar(kind, alpha), dA,
                                        A.ld, A.ld2, dB, B.ld, B.ld2, _dev_scalar(kind, beta), dC,
                                        C.ld, C.ld2, C.batch)
            assert rc == 0, tx.status_string(rc)
            torch.cuda.synchronize()
            got = dC.cpu().numpy()
            ref = run_oracle(kind, "N", "T", m, n, k, alpha, beta, A, B, C)
            if alpha == 0 or k == 0 or beta == 0:
                assert np.all(np.isfinite(C.dense(got))) or (beta == 1)
            C0 = C.dense()
            if (alpha == 0 or k == 0):
                # C <- beta*C exactly as the oracle (integer-free but single product per entry)
                assert np.allclose(C.dense(got).astype(np.complex128), C.dense(ref).astype(np.complex128),
                                   rtol=1e-6 if kind in "sc" else 1e-14, atol=0, equal_nan=True)
            else:
                check(kind, "N", "T", m, n, k, alpha, beta, A, B, C, got, ref)
            # same as the host-scalar call, bitwise (same kernels' arithmetic)
            if not (alpha == 0 or k == 0):
                rc2, got2, _ = run_lib(kind, "N", "T", m, n, k, alpha, beta, A, B, C)
                assert rc2 == 0
                assert np.array_equal(got.view(np.uint8), got2.view(np.uint8)), (m, n, k, alpha, beta)


@pytest.mark.parametrize("kind", "sdcz")
def test_device_alpha_beta_pointer_arrays(kind):
    import torch

    m, n, k = 8, 16, 4
    alpha, beta = _ab(kind, "devp")
    A, B, C = random_case(kind, m, n, k, 777, seed=42, tag="devp")
    dA, _ = to_dev(A)
    dB, _ = to_dev(B)
    dC, _ = to_dev(C)
    es = dA.element_size()
    perm = np.random.default_rng(5).permutation(C.batch)
    pa = torch.tensor(A.offsets()[perm] * es + dA.data_ptr(), device="cuda")
    pb = torch.tensor(B.offsets()[perm] * es + dB.data_ptr(), device="cuda")
    pc = torch.tensor(C.offsets()[perm] * es + dC.data_ptr(), device="cuda")
    rc = tx.tx_gemm_batched_ptr_dev(kind, "N", "N", m, n, k, _dev_scalar(kind, alpha), pa, A.ld,
                                    pb, B.ld, _dev_scalar(kind, beta), pc, C.ld, C.batch)
    assert rc == 0
    torch.cuda.synchronize()
    ref = run_oracle(kind, "N", "N", m, n, k, alpha, beta, A, B, C)
    check(kind, "N", "N", m, n, k, alpha, beta, A, B, C, dC.cpu().numpy(), ref)


def test_cuda_graph_capture_and_replay_with_device_scalars():
    """The calls only enqueue kernels on the given stream, so they can be captured in a
    CUDA graph (after a warm-up call has built any runtime-specialised instance).  With
    device-resident alpha/beta, the graph is replayed with new scalars, no re-capture."""
    import torch

    kind, n, batch = "d", 12, 5000
    A, B, C = random_case(kind, n, n, n, batch, seed=43, tag="graph")
    dA, _ = to_dev(A)
    dB, _ = to_dev(B)
    dC, _ = to_dev(C)
    C0 = dC.clone()
    da, db = _dev_scalar(kind, 0.5), _dev_scalar(kind, -0.25)
    s = torch.cuda.Stream()

    def call():
        assert tx.tx_gemm_batched_dev(kind, "T", "N", n, n, n, da, dA, n, n * n, dB, n, n * n, db,
                                      dC, n, n * n, batch, s) == 0
        assert tx.tx_gemm_batched(kind, "N", "N", n, n, n, 1.0, dA, n, n * n, dB, n, n * n, 1.0,
                                  dC, n, n * n, batch, s) == 0

    with torch.cuda.stream(s):
        call()  # warm-up (JIT instances, occupancy caches)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        call()
    for alpha, beta in ((0.5, -0.25), (2.0, 0.0), (0.0, 3.0)):
        dC.copy_(C0)
        da.fill_(alpha)
        db.fill_(beta)
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        got = dC.cpu().numpy()
        ref = C.buf.copy()
        assert oracle.gemm_batched(kind, "T", "N", n, n, n, alpha, A.buf, n, n * n, B.buf, n, n * n,
                                   beta, ref, n, n * n, batch) == 0
        C1 = Operand(kind, n, n, batch, 0)
        C1.buf[:] = ref
        ref2 = ref.copy()
        assert oracle.gemm_batched(kind, "N", "N", n, n, n, 1.0, A.buf, n, n * n, B.buf, n, n * n,
                                   1.0, ref2, n, n * n, batch) == 0
        # element-wise: the first call's error (<= tol * den1) passes into the second
        # with coefficient beta2 = 1, so the composite bound is tol * (den1 + den2)
        den1 = denominators(kind, "T", "N", alpha, beta, A, B, C.dense())
        den2 = denominators(kind, "N", "N", 1.0, 1.0, A, B, C1.dense())
        err = max_rel_err(kind, C.dense(got), C.dense(ref2), den1 + den2)
        assert err <= TOL[kind], (alpha, beta, err)


# --------------------------------------------------- sizes beyond 16 (NEXT-4)
@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("mnk", [(17, 17, 17), (24, 24, 24), (32, 32, 32), (32, 8, 20), (3, 32, 29),
                                 (48, 48, 48), (64, 64, 64), (64, 17, 40), (33, 64, 9)],
                         ids=lambda t: "x".join(map(str, t)))
def test_sizes_beyond_16(kind, mnk):
    """m, n, k up to 64 for s/d, 32 for c/z ("easily extended to larger sizes",
    PAPER.md:33-34): packed (runtime-specialised bulk), padded (gather) and both
    epilogues."""
    m, n, k = mnk
    if kind in "cz" and max(mnk) > 32:
        pytest.skip("c/z sizes stop at 32 (TX_MAX_DIM_CPLX)")
    ops = [("N", "N"), ("T", "N"), ("N", "C" if kind in "cz" else "T")]
    for ta, tb in ops:
        for general in (False, True):
            _case(kind, m, n, k, 211, ta, tb, general, "big")
    A, B, C = random_case(kind, m, n, k, 97, "T", "T", seed=44, tag="bigpad", pad=(1, 3),
                          c_sentinel=-1.5)
    alpha, beta = _ab(kind, "bigpad")
    rc, got, path = run_lib(kind, "T", "T", m, n, k, alpha, beta, A, B, C)
    assert rc == 0 and path[0] == "gather"
    ref = run_oracle(kind, "T", "T", m, n, k, alpha, beta, A, B, C)
    check(kind, "T", "T", m, n, k, alpha, beta, A, B, C, got, ref)


@pytest.mark.parametrize("kind,mnk", [("s", (51, 51, 51)), ("s", (63, 63, 63)), ("s", (57, 49, 61)),
                                      ("d", (63, 63, 63)), ("d", (49, 51, 53)), ("d", (37, 41, 43))],
                         ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
def test_odd_large_sizes_every_path(kind, mnk):
    """Odd sizes near the limit: two ring stages of one 16-byte alignment unit of pairs
    (4 pairs for s, 2 for d) exceed shared memory, so the packed CUDA-core path hands the
    batch to the gather kernels, whose stage regions are 16-byte aligned for any tile size
    (round 2 fix: these calls returned 'invalid argument').  Packed with the tensor-core
    kernel disabled, padded, and pointer arrays, each against the oracle."""
    import torch
    from paper_1304_7053_b200 import binding

    m, n, k = mnk
    prev = binding.set_tc(0)
    try:
        for ta, tb in (("N", "N"), ("T", "T")):
            for general in (False, True):
                _case(kind, m, n, k, 37, ta, tb, general, "oddbig")
                _case(kind, m, n, k, 29, ta, tb, general, "oddbigpad", pad=(1, 5))
        A, B, C = random_case(kind, m, n, k, 31, "N", "T", seed=12, tag="oddptr")
        alpha, beta = _ab(kind, "oddptr")
        dA, _ = to_dev(A)
        dB, _ = to_dev(B)
        dC, _ = to_dev(C)
        es = dA.element_size()
        perm = np.random.default_rng(3).permutation(C.batch)
        pa = torch.tensor(A.offsets()[perm] * es + dA.data_ptr(), device="cuda")
        pb = torch.tensor(B.offsets()[perm] * es + dB.data_ptr(), device="cuda")
        pc = torch.tensor(C.offsets()[perm] * es + dC.data_ptr(), device="cuda")
        rc = tx.tx_gemm_batched_ptr(kind, "N", "T", m, n, k, alpha, pa, A.ld, pb, B.ld, beta, pc,
                                    C.ld, C.batch)
        assert rc == 0, tx.status_string(rc)
        got = dC.cpu().numpy()
        ref = run_oracle(kind, "N", "T", m, n, k, alpha, beta, A, B, C)
        check(kind, "N", "T", m, n, k, alpha, beta, A, B, C, got, ref)
    finally:
        binding.set_tc(prev)


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("mnk", [(32, 32, 32), (24, 8, 32), (5, 30, 32), (64, 64, 64), (48, 40, 16)],
                         ids=lambda t: "x".join(map(str, t)))
def test_pointer_arrays_beyond_16(kind, mnk):
    """Pointer arrays at sizes 17-32 with k * sizeof(T) a multiple of 128 B (swizzled
    gather placement possible for op(A) = T/C and op(B) = N): permuted pointers,
    against the oracle and bitwise against the packed strided call."""
    import torch

    m, n, k = mnk
    if kind in "cz" and max(mnk) > 32:
        pytest.skip("c/z sizes stop at 32 (TX_MAX_DIM_CPLX)")
    for ta, tb in (("N", "N"), ("T", "N"), ("C" if kind in "cz" else "T", "T")):
        A, B, C = random_case(kind, m, n, k, 129, ta, tb, seed=12, tag="ptrbig")
        alpha, beta = _ab(kind, f"ptrbig{m}{n}{k}")
        rc, got_strided, spath = run_lib(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
        assert rc == 0
        perm = np.random.default_rng(6).permutation(C.batch)
        dA, _ = to_dev(A)
        dB, _ = to_dev(B)
        dC, _ = to_dev(C)
        es = dA.element_size()
        pa = torch.tensor(A.offsets()[perm] * es + dA.data_ptr(), device="cuda")
        pb = torch.tensor(B.offsets()[perm] * es + dB.data_ptr(), device="cuda")
        pc = torch.tensor(C.offsets()[perm] * es + dC.data_ptr(), device="cuda")
        rc = tx.tx_gemm_batched_ptr(kind, ta, tb, m, n, k, alpha, pa, A.ld, pb, B.ld, beta, pc,
                                    C.ld, C.batch)
        assert rc == 0
        got = dC.cpu().numpy()
        if spath[0] not in ("tc", "tc+tail"):  # the tensor-core kernel rounds differently
            assert np.array_equal(got.view(np.uint8), got_strided.view(np.uint8))
        ref = run_oracle(kind, ta, tb, m, n, k, alpha, beta, A, B, C)
        check(kind, ta, tb, m, n, k, alpha, beta, A, B, C, got, ref)


# ---------------------------------------------------------------- tx_prepare
@pytest.mark.parametrize("kind", "sdcz")
def test_prepare_builds_every_instance_the_call_uses(kind):
    """tx_prepare compiles/loads the runtime-specialised instances of a call shape; the
    call itself then compiles nothing, runs a runtime-specialised instance, and matches
    the oracle."""
    from paper_1304_7053_b200 import binding

    if binding.jit_compiled() < 0:
        pytest.skip("NVRTC unavailable")
    m, n, k = 11, 13, 6
    tb = "C" if kind in "cz" else "T"
    for layout, pad in (("packed", (0, 0)), ("strided", (1, 2))):
        for general in (False, True):
            assert tx.prepare(kind, "T", tb, m, n, k, beta_zero=not general, layout=layout) == 0
            before = binding.jit_compiled()
            err, path, _ = _case(kind, m, n, k, 2049, "T", tb, general, "prep", pad=pad)
            assert binding.jit_compiled() == before, (layout, general)
            assert binding.last_path_jit(), path
    # pointer arrays
    assert tx.prepare(kind, "N", "N", 9, 5, 7, beta_zero=False, layout="ptr") == 0
    before = binding.jit_compiled()
    import torch

    A, B, C = random_case(kind, 9, 5, 7, 500, seed=12, tag="prepptr")
    alpha, beta = _ab(kind, "prepptr")
    dA, _ = to_dev(A)
    dB, _ = to_dev(B)
    dC, _ = to_dev(C)
    Aa, Ba, Ca = (tx.pointer_array(x.view(500, -1).unsqueeze(2)) for x in (dA, dB, dC))
    tx.gemm_batched_ptr(Aa, Ba, Ca, 9, 5, 7, "N", "N", alpha, beta, dtype=dA.dtype)
    torch.cuda.synchronize()
    assert binding.jit_compiled() == before
    ref = run_oracle(kind, "N", "N", 9, 5, 7, alpha, beta, A, B, C)
    check(kind, "N", "N", 9, 5, 7, alpha, beta, A, B, C, dC.cpu().numpy(), ref)


def test_tensor_api_device_checks():
    import torch

    A = torch.zeros(4, 3, 3, device="cuda").transpose(1, 2)
    with pytest.raises(ValueError):
        tx.gemm_batched(A.cpu(), A, A.clone())
    pa = torch.zeros(4, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        tx.gemm_batched_ptr(pa, pa.cpu(), pa, 3, 3, 3, dtype=torch.float32)
    with pytest.raises(ValueError):
        tx.gemm_batched_ptr(pa, pa, pa.to(torch.int32), 3, 3, 3, dtype=torch.float32)


# ------------------------------------------- register-direct kernel (n <= 2)
@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("n", [1, 2])
def test_direct_tiny_matrices(kind, n):
    """Packed square n <= 2 runs the register-direct kernel (whole batch, including the
    batch % G tail pairs): against the oracle, and bitwise against the pointer-array
    path (a different kernel with the same ascending-l FMA chain and epilogue); beta == 0
    never reads C (NaN-filled)."""
    import torch

    for batch in (1, 3, 5, 1001, 65537):
        for ta, tb in ops_for(kind)[:4] + ops_for(kind)[-1:]:
            for general in (False, True):
                A, B, C = random_case(kind, n, n, n, batch, ta, tb, seed=71, tag="direct")
                if not general:
                    C.buf[:] = np.nan
                alpha, beta = _ab(kind, f"direct{n}{ta}{tb}", general)
                rc, got, path = run_lib(kind, ta, tb, n, n, n, alpha, beta, A, B, C)
                assert rc == 0 and path == ("direct", 1), path
                ref = run_oracle(kind, ta, tb, n, n, n, alpha, beta, A, B, C)
                check(kind, ta, tb, n, n, n, alpha, beta, A, B, C, got, ref)
                dA, _ = to_dev(A)
                dB, _ = to_dev(B)
                dC, _ = to_dev(C)
                es = dA.element_size()
                pa = torch.tensor(A.offsets() * es + dA.data_ptr(), device="cuda")
                pb = torch.tensor(B.offsets() * es + dB.data_ptr(), device="cuda")
                pc = torch.tensor(C.offsets() * es + dC.data_ptr(), device="cuda")
                assert tx.tx_gemm_batched_ptr(kind, ta, tb, n, n, n, alpha, pa, n, pb, n, beta, pc,
                                              n, batch) == 0
                assert np.array_equal(dC.cpu().numpy().view(np.uint8), got.view(np.uint8))


# -------------------------------------------- FP64 tensor cores (DMMA), d / z
@pytest.mark.parametrize("kind", "dz")
@pytest.mark.parametrize("n", range(1, 17))
def test_dmma_square_instances_bitwise_vs_fma_path(kind, n):
    """Square d/z instances run the FP64 tensor cores (mma.sync m8n8k4, one warp per
    pair); the generic AOT pointer-array kernel (runtime specialisation off) runs the
    FMA micro-tiles.  DMMA is the same fused FMA chain over k (tools/dmma_probe.py),
    so the two are bitwise equal; both match the oracle.  Ragged batches, every op
    pair, both epilogues."""
    import torch
    from paper_1304_7053_b200 import binding

    for ta, tb in ops_for(kind):
        for general in (False, True):
            err, path, (A, B, C, alpha, beta, got, ref) = _case(kind, n, n, n, 999, ta, tb, general,
                                                                f"dmma{n}")
            dA, _ = to_dev(A)
            dB, _ = to_dev(B)
            dC, _ = to_dev(C)
            es = dA.element_size()
            pa = torch.tensor(A.offsets() * es + dA.data_ptr(), device="cuda")
            pb = torch.tensor(B.offsets() * es + dB.data_ptr(), device="cuda")
            pc = torch.tensor(C.offsets() * es + dC.data_ptr(), device="cuda")
            prev = binding.set_jit(False)
            try:
                assert tx.tx_gemm_batched_ptr(kind, ta, tb, n, n, n, alpha, pa, A.ld, pb, B.ld,
                                              beta, pc, C.ld, C.batch) == 0
                assert not binding.last_path_jit()
            finally:
                binding.set_jit(prev)
            assert np.array_equal(dC.cpu().numpy().view(np.uint8), got.view(np.uint8)), (n, ta, tb)
