"""Replays of the paper's experiments (§8.1-8.5, Figs. 2-9, Table 1) on one B200,
with this library.  Writes one JSON object per experiment.

  fig2_grid     -- throughput vs number of CTAs (the paper's block-count sweep)
  fig3_batch    -- throughput vs batch size 10^3..10^7
  fig4_ops      -- c64, all 9 op pairs, general alpha/beta, ratio to N/N
  fig5_beta0    -- s, a1b0 (alpha=1, beta=0) vs general alpha/beta, n = 1..16
  table1        -- GFlop/s for 10^5 pairs, n = 1..16, 4 types, a1b0
  fig7_iface    -- strided vs pointer-array vs cuBLAS strided-batched (torch.baddbmm,
                   context only), s and c, a1b0
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1304_7053_b200 as tx  # noqa: E402
import txinputs  # noqa: E402
from paper_1304_7053_b200 import model  # noqa: E402

TD = {"s": torch.float32, "d": torch.float64, "c": torch.complex64, "z": torch.complex128}


def data(kind, n, batch, r=0):
    key = lambda nm: txinputs.stream_key(5, "exp", kind, n, r, nm)
    return [txinputs.values_torch(kind, key(nm), 0, n * n * batch, "cuda") for nm in "ABC"]


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]  # median (the paper's protocol)


def gemm(kind, n, batch, A, B, C, alpha, beta, ta="N", tb="N"):
    rc = tx.tx_gemm_batched(kind, ta, tb, n, n, n, alpha, A, n, n * n, B, n, n * n, beta, C, n,
                            n * n, batch)
    assert rc == 0


def gflops(kind, n, batch, ms):
    return round(model.flops(kind, n, n, n, batch) / (ms / 1e3) / 1e9, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    out = open(a.out, "w")
    only = set(a.only.split(",")) if a.only else None

    def emit(d):
        out.write(json.dumps(d) + "\n")
        out.flush()
        print(d["experiment"], "done", file=sys.stderr, flush=True)

    if not only or "fig2_grid" in only:
        rows = []
        for n in (4, 10, 16):
            A, B, C = data("s", n, 100_000)
            for g in (1, 8, 37, 74, 148, 296, 592, 2000, 0):
                tx.set_max_ctas(g)
                ms = timeit(lambda: gemm("s", n, 100_000, A, B, C, 0.5, 0.25))
                rows.append({"n": n, "ctas": g or "auto", "gflops": gflops("s", n, 100_000, ms)})
            tx.set_max_ctas(0)
        emit({"experiment": "fig2_grid", "kind": "s", "batch": 100_000, "rows": rows,
              "cite": "PAPER.md:579-587 (more than 2000 blocks: very little to gain on K20c)"})
    if not only or "fig3_batch" in only:
        rows = []
        for n in (4, 10, 16):
            for batch in (1_000, 2_000, 10_000, 100_000, 1_000_000, 10_000_000):
                A, B, C = data("s", n, batch)
                ms = timeit(lambda: gemm("s", n, batch, A, B, C, 0.5, 0.25), reps=5)
                rows.append({"n": n, "batch": batch, "gflops": gflops("s", n, batch, ms),
                             "us": round(ms * 1e3, 2)})
                del A, B, C
                torch.cuda.empty_cache()
        emit({"experiment": "fig3_batch", "kind": "s", "rows": rows,
              "cite": "PAPER.md:587-597 (gains grow slowly with batch; 2000 not much worse)"})
    if not only or "fig4_ops" in only:
        rows = []
        for n in range(1, 17):
            A, B, C = data("c", n, 100_000)
            base = None
            for ta in "NTC":
                for tb in "NTC":
                    ms = timeit(lambda: gemm("c", n, 100_000, A, B, C, 0.5 + 0.25j, 0.3 - 0.1j,
                                             ta, tb))
                    g = gflops("c", n, 100_000, ms)
                    base = g if ta + tb == "NN" else base
                    rows.append({"n": n, "ops": ta + tb, "gflops": g, "ratio_to_NN": round(g / base, 3)})
        emit({"experiment": "fig4_ops", "kind": "c", "batch": 100_000, "rows": rows,
              "cite": "PAPER.md:617-634 (conj/transpose slowdown 'minor')"})
    if not only or "fig5_beta0" in only:
        rows = []
        for n in range(1, 17):
            A, B, C = data("s", n, 100_000)
            t0 = timeit(lambda: gemm("s", n, 100_000, A, B, C, 1.0, 0.0))
            t1 = timeit(lambda: gemm("s", n, 100_000, A, B, C, 0.5, 0.25))
            rows.append({"n": n, "a1b0_gflops": gflops("s", n, 100_000, t0),
                         "general_gflops": gflops("s", n, 100_000, t1), "gain": round(t1 / t0, 3)})
        emit({"experiment": "fig5_beta0", "kind": "s", "batch": 100_000, "rows": rows,
              "cite": "PAPER.md:636-655 (a1b0 gain 10-50% on K20c); bytes 3 vs 4 matrices"})
    if not only or "table1" in only:
        rows = []
        for kind in "sdcz":
            for n in range(1, 17):
                A, B, C = data(kind, n, 100_000)
                ms = timeit(lambda: gemm(kind, n, 100_000, A, B, C, 1.0, 0.0))
                rows.append({"kind": kind, "n": n, "gflops": gflops(kind, n, 100_000, ms)})
        emit({"experiment": "table1", "batch": 100_000, "mode": "a1b0", "rows": rows,
              "paper_k20c": {"s": [1, 3, 12, 26, 48, 59, 83, 125, 102, 104, 126, 129, 124, 126, 150, 216],
                             "d": [1, 4, 11, 17, 39, 48, 68, 86, 86, 90, 110, 122, 114, 115, 131, 173],
                             "c": [2, 10, 42, 87, 143, 187, 263, 327, 334, 362, 439, 480, 446, 436, 504, 609],
                             "z": [2, 9, 34, 52, 102, 100, 146, 204, 127, 149, 172, 186, 172, 177, 212, 217]},
              "cite": "PAPER.md:742-771 (Table 1, K20c) -- context only"})
    if not only or "fig7_iface" in only:
        rows = []
        for kind in "sc":
            for n in (2, 4, 8, 10, 16):
                batch = 100_000
                A, B, C = data(kind, n, batch)
                e = A.element_size()
                pa = A.data_ptr() + torch.arange(batch, device="cuda") * (n * n * e)
                pb = B.data_ptr() + torch.arange(batch, device="cuda") * (n * n * e)
                pc = C.data_ptr() + torch.arange(batch, device="cuda") * (n * n * e)
                t_u = timeit(lambda: gemm(kind, n, batch, A, B, C, 1.0, 0.0))
                t_p = timeit(lambda: tx.tx_gemm_batched_ptr(kind, "N", "N", n, n, n, 1.0, pa, n, pb,
                                                            n, 0.0, pc, n, batch))
                # cuBLAS strided-batched through torch (column-major = transposed row-major)
                At = A.view(batch, n, n)
                Bt = B.view(batch, n, n)
                Ct = C.view(batch, n, n)
                t_c = timeit(lambda: torch.bmm(Bt, At, out=Ct))
                rows.append({"kind": kind, "n": n, "unif_gflops": gflops(kind, n, batch, t_u),
                             "nounif_gflops": gflops(kind, n, batch, t_p),
                             "cublas_bmm_gflops": gflops(kind, n, batch, t_c),
                             "unif_over_nounif": round(t_p / t_u, 3),
                             "unif_over_cublas": round(t_c / t_u, 3)})
        emit({"experiment": "fig7_iface", "mode": "a1b0", "batch": 100_000, "rows": rows,
              "cite": "PAPER.md:679-740 (unif vs nounif vs cuBLAS); cuBLAS 12.x here is context"})


if __name__ == "__main__":
    main()
