"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Inputs are generated on the device from the same counter-based streams the host
generator produces (txinputs); outputs are checked on sampled pairs the oracle
recomputes one by one (first, last and seeded random pairs).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1304_7053_b200 as tx
import txinputs
from helpers import TOL, WIDE, Operand, max_rel_err

pytestmark = pytest.mark.gpu


def dev_batch(kind, rows, cols, batch, key):
    return txinputs.values_torch(kind, key, 0, rows * cols * batch, "cuda")


def sample_idx(batch, count, seed):
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, batch - 1], rng.integers(0, batch, count)]))
    return idx


def sampled_check(kind, ta, tb, m, n, k, alpha, beta, dA, dB, dC0_samples, dC, idx):
    import torch

    ra, ca = (m, k) if ta in "nN" else (k, m)
    rb, cb = (k, n) if tb in "nN" else (n, k)
    ti = torch.as_tensor(idx, device=dA.device)
    hA = dA.view(-1, ra * ca)[ti].cpu().numpy().ravel()
    hB = dB.view(-1, rb * cb)[ti].cpu().numpy().ravel()
    hC = dC0_samples.copy()
    got = dC.view(-1, m * n)[ti].cpu().numpy().ravel()
    s = len(idx)
    rc = oracle.gemm_batched(kind, ta, tb, m, n, k, alpha, hA, ra, ra * ca, hB, rb, rb * cb, beta,
                             hC, m, m * n, s)
    assert rc == 0
    # error denominators on the sample
    Ad = hA.reshape(s, ca, ra).transpose(0, 2, 1).astype(WIDE[kind])
    Bd = hB.reshape(s, cb, rb).transpose(0, 2, 1).astype(WIDE[kind])
    if ta not in "nN":
        Ad = Ad.transpose(0, 2, 1)
    if tb not in "nN":
        Bd = Bd.transpose(0, 2, 1)
    den = abs(alpha) * np.einsum("pil,plj->pij", np.abs(Ad), np.abs(Bd))
    if beta != 0:
        den = den + abs(beta) * np.abs(dC0_samples.reshape(s, n, m).transpose(0, 2, 1))
    err = max_rel_err(kind, got.reshape(s, n, m).transpose(0, 2, 1),
                      hC.reshape(s, n, m).transpose(0, 2, 1), den)
    assert err <= TOL[kind], err
    return err


def run_full(kind, m, n, k, batch, ta="N", tb="N", general=True, samples=4096, seed=1):
    import torch

    key = lambda name: txinputs.stream_key(txinputs.DEFAULT_SEED, "full", kind, m, n, k, name)
    dA = dev_batch(kind, m, k, batch, key("A"))
    dB = dev_batch(kind, k, n, batch, key("B"))
    dC = dev_batch(kind, m, n, batch, key("C"))
    alpha = txinputs.scalar(kind, key("alpha"))
    beta = txinputs.scalar(kind, key("beta")) if general else 0
    idx = sample_idx(batch, samples, seed)
    C0 = dC.view(-1, m * n)[torch.as_tensor(idx, device="cuda")].cpu().numpy().ravel()
    rc = tx.tx_gemm_batched(kind, ta, tb, m, n, k, alpha, dA, m if ta in "nN" else k,
                            m * k, dB, k if tb in "nN" else n, k * n, beta, dC, m, m * n, batch)
    assert rc == 0, tx.status_string(rc)
    path = tx.last_path()
    torch.cuda.synchronize()
    err = sampled_check(kind, ta, tb, m, n, k, alpha, beta, dA, dB, C0, dC, idx)
    del dA, dB, dC
    torch.cuda.empty_cache()
    return err, path


@pytest.mark.parametrize("n", [10, 16])
def test_config2_sgemm_100k_general(n):
    """BASELINE configs[1]: SGEMM 100,000 pairs, n = 10 and 16, N/N, general alpha/beta
    -- the bench workload.  All 100,000 pairs are checked."""
    err, path = run_full("s", n, n, n, 100_000, samples=100_000)
    assert path[0] == "bulk"


def test_config1_small():
    """BASELINE configs[0]: 1,000 4x4 SGEMM pairs, alpha = 1, beta = 0, fully checked."""
    import torch

    kind, n, batch = "s", 4, 1000
    key = lambda name: txinputs.stream_key(txinputs.DEFAULT_SEED, "cfg1", name)
    dA = dev_batch(kind, n, n, batch, key("A"))
    dB = dev_batch(kind, n, n, batch, key("B"))
    dC = torch.full((n * n * batch,), float("nan"), device="cuda")
    assert tx.tx_gemm_batched(kind, "N", "N", n, n, n, 1.0, dA, n, n * n, dB, n, n * n, 0.0, dC,
                              n, n * n, batch) == 0
    torch.cuda.synchronize()
    hA, hB = dA.cpu().numpy(), dB.cpu().numpy()
    hC = np.full(n * n * batch, np.nan, dtype=np.float32)
    assert oracle.gemm_batched(kind, "N", "N", n, n, n, 1.0, hA, n, n * n, hB, n, n * n, 0.0, hC,
                               n, n * n, batch) == 0
    got = dC.cpu().numpy()
    den = np.einsum("pil,plj->pij", np.abs(hA.reshape(batch, n, n).transpose(0, 2, 1)),
                    np.abs(hB.reshape(batch, n, n).transpose(0, 2, 1)).astype(np.float64))
    err = max_rel_err(kind, got.reshape(batch, n, n), hC.reshape(batch, n, n),
                      den.transpose(0, 2, 1))
    assert err <= TOL[kind]


OPS = {"s": "NT", "d": "NT", "c": "NTC", "z": "NTC"}


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("n", range(1, 17))
def test_config3_all_ops_1e5_sampled(kind, n):
    """BASELINE configs[2] at its real size: 100,000 pairs for every type, n = 1..16,
    every op pair and both epilogues, in the
    launch configuration the sweep times (automatic grid, many tiles per CTA)."""
    for ta in OPS[kind]:
        for tb in OPS[kind]:
            for general in (False, True):
                err, path = run_full(kind, n, n, n, 100_000, ta, tb, general, samples=256,
                                     seed=n)
                assert path[0] == ("direct" if n <= 2 else "bulk"), path


@pytest.mark.parametrize("kind", "sdcz")
def test_gate_size_1e6_sampled(kind):
    """North-star gate workload: 10^6 pairs of 16x16, beta == 0 and general."""
    for general in (False, True):
        run_full(kind, 16, 16, 16, 1_000_000, general=general, samples=2048)


@pytest.mark.parametrize("kind", "dz")
def test_config5_1e7_sampled(kind):
    """BASELINE configs[4]: D/Z 16x16 with 10^7 pairs (one GPU's worth at G = 1)."""
    import torch

    free, _ = torch.cuda.mem_get_info()
    need = 3 * 10_000_000 * 256 * (8 if kind == "d" else 16) + (1 << 30)
    if free < need:
        pytest.skip(f"needs {need / 1e9:.0f} GB free")
    run_full(kind, 16, 16, 16, 10_000_000, general=True, samples=4096)


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("mnk", [(8, 16, 4), (16, 3, 16)], ids=lambda t: "x".join(map(str, t)))
def test_config4_pointer_1e6_sampled(kind, mnk):
    """BASELINE configs[3]: non-square, pointer-array layout, 10^6 pairs, pointers in a
    seeded random order."""
    import torch

    m, n, k = mnk
    batch = 1_000_000
    key = lambda name: txinputs.stream_key(txinputs.DEFAULT_SEED, "cfg4", kind, m, n, k, name)
    dA = dev_batch(kind, m, k, batch, key("A"))
    dB = dev_batch(kind, k, n, batch, key("B"))
    dC = dev_batch(kind, m, n, batch, key("C"))
    alpha, beta = txinputs.scalar(kind, key("alpha")), txinputs.scalar(kind, key("beta"))
    perm = torch.as_tensor(np.random.default_rng(3).permutation(batch), device="cuda")
    es = dA.element_size()
    pa = dA.data_ptr() + perm * (m * k * es)
    pb = dB.data_ptr() + perm * (k * n * es)
    pc = dC.data_ptr() + perm * (m * n * es)
    idx = sample_idx(batch, 2048, 4)
    C0 = dC.view(-1, m * n)[torch.as_tensor(idx, device="cuda")].cpu().numpy().ravel()
    rc = tx.tx_gemm_batched_ptr(kind, "N", "N", m, n, k, alpha, pa, m, pb, k, beta, pc, m, batch)
    assert rc == 0 and tx.last_path()[0] == "ptr"
    torch.cuda.synchronize()
    sampled_check(kind, "N", "N", m, n, k, alpha, beta, dA, dB, C0, dC, idx)
