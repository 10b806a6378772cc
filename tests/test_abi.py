"""The C-ABI library builds, loads and exports every symbol include/txgemm.h
declares; argument validation is pure host code (no GPU needed) and returns the
same codes as the oracle's independent validation."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_1304_7053_b200 as tx
from paper_1304_7053_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "txgemm.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tx_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    L = tx.lib()
    syms = declared_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(L, s), s


def test_version_and_instances():
    assert tx.version() == 10100
    assert tx.num_instances() > 800
    assert "success" in tx.status_string(0)
    assert "lda" in tx.status_string(-8)


def test_no_fallback_when_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(binding, "_lib", None)
    monkeypatch.setattr(binding, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError):
        binding.lib()


# Invalid argument vectors: the library's host validation must agree with the
# oracle's independent re-implementation.  No device memory is touched because
# every vector fails validation (fake, never-dereferenced addresses).
FAKE = 1 << 40


def _vec(**kw):
    d = dict(ta="N", tb="N", m=4, n=4, k=4, alpha=1.0, lda=4, lda2=16, ldb=4, ldb2=16, beta=0.0,
             ldc=4, ldc2=16, batch=3, alpha_ptr=True, beta_ptr=True, A=FAKE, B=FAKE + (1 << 20),
             C=FAKE + (2 << 20))
    d.update(kw)
    return d


BAD = [
    dict(ta="x"), dict(tb="?"), dict(m=-1), dict(m=65), dict(n=99), dict(k=-3),
    dict(alpha_ptr=False), dict(beta_ptr=False), dict(lda=3), dict(ta="T", k=5, lda=4),
    dict(ldb=2), dict(ldc=1), dict(lda2=-5), dict(ldb2=-1), dict(ldc2=15), dict(batch=-2),
    dict(A=None), dict(B=None), dict(C=None), dict(C=FAKE + 8),  # C overlaps A
    dict(C=FAKE + (1 << 20) + 40),  # C overlaps B
    dict(A=FAKE + 2), dict(B=FAKE + (1 << 20) + 2), dict(C=FAKE + (2 << 20) + 2),  # misaligned
]


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("i", range(len(BAD)))
def test_validation_matches_oracle(kind, i):
    v = _vec(**BAD[i])
    es = {"s": 4, "d": 8, "c": 8, "z": 16}[kind]
    got = tx.tx_gemm_batched(kind, v["ta"], v["tb"], v["m"], v["n"], v["k"], v["alpha"], v["A"],
                             v["lda"], v["lda2"], v["B"], v["ldb"], v["ldb2"], v["beta"], v["C"],
                             v["ldc"], v["ldc2"], v["batch"], stream=0, alpha_ptr=v["alpha_ptr"],
                             beta_ptr=v["beta_ptr"])
    assert got < 0
    # oracle on host buffers laid out at the same relative offsets
    base = np.zeros((3 << 20) // es + 64, dtype=oracle.NP_DTYPE[kind])

    def off(x):
        return None if x is None else (x - FAKE) // es

    want = oracle.lib()  # noqa: F841 (ensure built)
    want = getattr(oracle.lib(), f"oracle_gemm_batched_{kind}")(
        v["ta"].encode(), v["tb"].encode(), v["m"], v["n"], v["k"],
        ctypes.addressof(oracle._scalar(kind, v["alpha"])) if v["alpha_ptr"] else None,
        None if v["A"] is None else base.ctypes.data + (v["A"] - FAKE), v["lda"], v["lda2"],
        None if v["B"] is None else base.ctypes.data + (v["B"] - FAKE), v["ldb"], v["ldb2"],
        ctypes.addressof(oracle._scalar(kind, v["beta"])) if v["beta_ptr"] else None,
        None if v["C"] is None else base.ctypes.data + (v["C"] - FAKE), v["ldc"], v["ldc2"],
        v["batch"])
    assert got == want, (BAD[i], got, want)


@pytest.mark.parametrize("kind", "sdcz")
def test_ptr_validation_codes(kind):
    f = tx.tx_gemm_batched_ptr
    assert f(kind, "N", "N", 2, 2, 2, 1, FAKE, 2, FAKE, 2, 0, FAKE, 2, 1, 0, beta_ptr=False) == -11
    assert f(kind, "N", "N", 2, 2, 2, 1, FAKE, 2, FAKE, 1, 0, FAKE, 2, 1, 0) == -10
    assert f(kind, "N", "N", 2, 2, 2, 1, FAKE, 2, FAKE, 2, 0, FAKE, 1, 1, 0) == -13
    assert f(kind, "N", "N", 2, 2, 2, 1, FAKE, 2, FAKE, 2, 0, FAKE, 2, -1, 0) == -14
    assert f(kind, "N", "N", 2, 2, 2, 1, FAKE, 2, None, 2, 0, FAKE, 2, 1, 0) == -9
    assert f(kind, "N", "N", 2, 2, 2, 1, FAKE, 2, FAKE, 2, 0, None, 2, 1, 0) == -12
    assert f(kind, "N", "N", 2, 2, 2, 1, None, 2, FAKE, 2, 0, FAKE, 2, 1, 0) == -7


@pytest.mark.parametrize("kind", "sdcz")
def test_quick_returns_launch_nothing(kind):
    """m == 0, batch == 0 and (alpha == 0, beta == 1) return 0 without any CUDA call
    (works with no GPU present)."""
    f = tx.tx_gemm_batched
    assert f(kind, "N", "N", 0, 4, 4, 1, FAKE, 1, 0, FAKE, 4, 16, 0, FAKE, 1, 4, 5, stream=0) == 0
    assert tx.last_path() == ("none", 0)
    assert f(kind, "N", "N", 4, 4, 4, 1, FAKE, 4, 16, FAKE + (1 << 20), 4, 16, 0, FAKE + (2 << 20),
             4, 16, 0, stream=0) == 0
    assert f(kind, "N", "N", 4, 4, 4, 0, None, 4, 16, None, 4, 16, 1, FAKE, 4, 16, 3, stream=0) == 0
    assert f(kind, "N", "N", 4, 4, 0, 2, None, 4, 16, None, 4, 16, 1, FAKE, 4, 16, 3, stream=0) == 0


def test_hostio_staging_checks():
    f = tx.tx_gemm_batched_hostio
    h = np.zeros(64, dtype=np.float32)
    hp = h.ctypes.data
    assert f("s", "N", "N", 2, 2, 2, 1, hp, 2, 4, hp + 64, 2, 4, 0, hp + 128, 2, 4, 2, 0, None,
             FAKE, FAKE) == -19
    assert f("s", "N", "N", 2, 2, 2, 1, hp, 2, 4, hp + 64, 2, 4, 0, hp + 128, 2, 4, 2, 0, FAKE,
             None, FAKE) == -20
    assert f("s", "N", "N", 2, 2, 2, 1, hp, 2, 4, hp + 64, 2, 4, 0, hp + 128, 2, 4, 2, 0, FAKE,
             FAKE, None) == -21


def test_z_needs_16_byte_alignment():
    """tx_cdouble matrices 8-byte aligned (legal for the C struct) are rejected: the
    kernels move 16-byte elements (R21)."""
    f = tx.tx_gemm_batched
    assert f("z", "N", "N", 4, 4, 4, 1, FAKE + 8, 4, 16, FAKE + (1 << 20), 4, 16, 0,
             FAKE + (2 << 20), 4, 16, 3, stream=0) == -7
    assert f("z", "N", "N", 4, 4, 4, 1, FAKE, 4, 16, FAKE + (1 << 20) + 8, 4, 16, 0,
             FAKE + (2 << 20), 4, 16, 3, stream=0) == -10
    assert f("z", "N", "N", 4, 4, 4, 1, FAKE, 4, 16, FAKE + (1 << 20), 4, 16, 0,
             FAKE + (2 << 20) + 8, 4, 16, 3, stream=0) == -14
    # pointer arrays must be 8-byte aligned
    g = tx.tx_gemm_batched_ptr
    assert g("d", "N", "N", 2, 2, 2, 1, FAKE + 4, 2, FAKE, 2, 0, FAKE, 2, 1, 0) == -7
    assert g("d", "N", "N", 2, 2, 2, 1, FAKE, 2, FAKE + 4, 2, 0, FAKE, 2, 1, 0) == -9
    assert g("d", "N", "N", 2, 2, 2, 1, FAKE, 2, FAKE, 2, 0, FAKE + 4, 2, 1, 0) == -12
    # host-buffer staging buffers likewise
    h = tx.tx_gemm_batched_hostio
    hb = np.zeros(4096, dtype=np.complex128)
    hp = (hb.ctypes.data + 63) // 64 * 64
    assert h("z", "N", "N", 2, 2, 2, 1, hp, 2, 4, hp + 1024, 2, 4, 0, hp + 2048, 2, 4, 2, 0,
             FAKE + 8, FAKE, FAKE) == -19


def test_prepare_argument_errors():
    """tx_prepare validates before touching the device (no GPU needed)."""
    assert tx.prepare("q", "N", "N", 4, 4, 4) == -1
    assert tx.prepare("s", "x", "N", 4, 4, 4) == -2
    assert tx.prepare("d", "N", "?", 4, 4, 4) == -3
    assert tx.prepare("c", "N", "N", 33, 4, 4) == -4
    assert tx.prepare("z", "N", "N", 4, -1, 4) == -5
    assert tx.prepare("s", "N", "N", 4, 4, 99) == -6
    assert tx.prepare("s", "N", "N", 4, 4, 4, layout=7) == -8
    assert tx.prepare("s", "N", "N", 0, 4, 4) == 0  # quick return: nothing to build


def test_complex_size_limit():
    """m, n, k up to 64 for s/d but 32 for c/z (include/txgemm.h TX_MAX_DIM_CPLX)."""
    f = tx.tx_gemm_batched
    for kind in "cz":
        assert f(kind, "N", "N", 33, 4, 4, 1, FAKE, 33, 132, FAKE + (1 << 20), 4, 16, 0,
                 FAKE + (2 << 20), 33, 132, 3, stream=0) == -3
        assert f(kind, "N", "N", 4, 33, 4, 1, FAKE, 4, 16, FAKE + (1 << 20), 4, 132, 0,
                 FAKE + (2 << 20), 4, 132, 3, stream=0) == -4
        assert f(kind, "N", "N", 4, 4, 33, 1, FAKE, 4, 132, FAKE + (1 << 20), 33, 132, 0,
                 FAKE + (2 << 20), 4, 16, 3, stream=0) == -5
    for kind in "sd":  # 65 is past the real limit
        assert f(kind, "N", "N", 65, 4, 4, 1, FAKE, 65, 260, FAKE + (1 << 20), 4, 16, 0,
                 FAKE + (2 << 20), 65, 260, 3, stream=0) == -3
