"""Gate sweep (north star): every type x n = 1..16, N/N (and optionally all ops), beta == 0
and general, at 10^6 pairs per GPU; algorithmic GB/s and % of the measured HBM peak.

Sustained protocol: back-to-back launches over R rotating buffer sets whose
total footprint is >= 4 x L2, so no set is L2-resident when it is reused.
Writes one JSON line per case to stdout (and --out)."""
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

L2 = 126 * 1024 * 1024

try:  # SM clock / power-cap state sampled while the timed calls run
    import pynvml

    pynvml.nvmlInit()
    _NVH = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # pragma: no cover - no NVML
    _NVH = None


def _clock_sample():
    if _NVH is None:
        return None
    try:
        mhz = pynvml.nvmlDeviceGetClockInfo(_NVH, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(_NVH)
        return {"sm_mhz": mhz, "power_cap": bool(r & pynvml.nvmlClocksEventReasonSwPowerCap)}
    except Exception:
        return None


def run_case(kind, m, n, k, batch, ta, tb, general, reps, peak, layout="strided", graph=False):
    es = model.ESIZE[kind]
    per_set = es * (m * k + k * n + m * n) * batch
    ptr = layout == "ptr"
    shA, shB = layout == "sharedA", layout == "sharedB"
    R = max(1, min(64, -(-4 * L2 // per_set)))
    sets = []
    for r in range(R):
        key = lambda nm: txinputs.stream_key(7, "sweep", kind, m, n, k, r, nm)
        A = txinputs.values_torch(kind, key("A"), 0, m * k * batch, "cuda")
        B = txinputs.values_torch(kind, key("B"), 0, k * n * batch, "cuda")
        C = txinputs.values_torch(kind, key("C"), 0, m * n * batch, "cuda")
        sets.append((A, B, C))
    alpha = txinputs.scalar(kind, 11)
    beta = txinputs.scalar(kind, 12) if general else 0
    lda = m if ta in "nN" else k
    ldb = k if tb in "nN" else n

    if ptr:  # pointer arrays in a seeded random order (BASELINE configs[3])
        perm = torch.randperm(batch, generator=torch.Generator().manual_seed(3)).cuda()
        psets = []
        for A, B, C in sets:
            e = A.element_size()
            psets.append((A.data_ptr() + perm * (m * k * e), B.data_ptr() + perm * (k * n * e),
                          C.data_ptr() + perm * (m * n * e)))

    def call(i):
        s = sets[i]
        if ptr:
            pa, pb, pc = psets[i]
            rc = tx.tx_gemm_batched_ptr(kind, ta, tb, m, n, k, alpha, pa, lda, pb, ldb, beta, pc,
                                        m, batch)
        else:
            A, B, C = s
            rc = tx.tx_gemm_batched(kind, ta, tb, m, n, k, alpha, A, lda, 0 if shA else m * k, B,
                                    ldb, 0 if shB else k * n, beta, C, m, m * n, batch)
        assert rc == 0, tx.status_string(rc)

    for i in range(2 * R):
        call(i % R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        call(i % R)
    e1.record()
    clk = _clock_sample()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ms_stream = ms
    if graph:
        # Device-side rate without the host's per-call cost: the same `reps` calls
        # captured once into a CUDA graph (PDL edges kept) and replayed.
        g = torch.cuda.CUDAGraph()
        s_cap = torch.cuda.Stream()
        with torch.cuda.stream(s_cap):
            with torch.cuda.graph(g, stream=s_cap):
                for i in range(reps):
                    call(i % R)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        clk = _clock_sample()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    byts = model.bytes_moved(kind, m, n, k, batch, True, general, shared_a=shA, shared_b=shB)
    if ptr:
        byts_ptr = model.bytes_moved(kind, m, n, k, batch, True, general, pointer_arrays=True)
    gbps = byts / (ms / 1e3) / 1e9
    return {"kind": kind, "m": m, "n": n, "k": k, "ops": ta + tb, "beta0": not general,
            "batch": batch, "us": round(ms * 1e3, 2), "gbps": round(gbps, 1),
            "frac_measured": round(gbps / peak, 4),
            "gflops": round(model.flops(kind, m, n, k, batch) / (ms / 1e3) / 1e9, 1),
            "path": tx.last_path()[0], "sets": R, "layout": layout, "clock": clk,
            **({"timing": "cuda graph of back-to-back calls", "us_stream": round(ms_stream * 1e3, 2)}
               if graph else {}),
            **({"gbps_with_pointers": round(byts_ptr / (ms / 1e3) / 1e9, 1)} if ptr else {})}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="sdcz")
    ap.add_argument("--sizes", default="1-16")
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--ops", default="NN")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    ap.add_argument("--shapes", default="", help="m x n x k list, e.g. 8x16x4,16x3x16")
    ap.add_argument("--graph", action="store_true",
                    help="time a CUDA-graph replay of the calls (device time, no host launch cost)")
    ap.add_argument("--layout", default="strided", choices=("strided", "ptr", "sharedA", "sharedB"))
    a = ap.parse_args()
    lo, hi = (int(x) for x in a.sizes.split("-")) if "-" in a.sizes else (int(a.sizes),) * 2
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = open(a.out, "w") if a.out else None
    ops = a.ops.split(",")
    if a.shapes:
        for kind in a.kinds:
            for shp in a.shapes.split(","):
                m, n, k = (int(x) for x in shp.split("x"))
                for op in ops:
                    if kind in "sd" and "C" in op:
                        continue
                    for general in (False, True):
                        r = run_case(kind, m, n, k, a.batch, op[0], op[1], general, a.reps, peak,
                                     a.layout, a.graph)
                        print(json.dumps(r), flush=True)
                        if out:
                            out.write(json.dumps(r) + "\n")
                        torch.cuda.empty_cache()
        return
    for kind in a.kinds:
        for nn in range(lo, hi + 1):
            for op in ops:
                if kind in "sd" and "C" in op:
                    continue
                for general in (False, True):
                    r = run_case(kind, nn, nn, nn, a.batch, op[0], op[1], general, a.reps, peak,
                                 graph=a.graph)
                    line = json.dumps(r)
                    print(line, flush=True)
                    if out:
                        out.write(line + "\n")
                    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
