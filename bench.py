#!/usr/bin/env python
"""Benchmark of the batched small-matrix GEMM hot path (BASELINE.json).

Workload (BASELINE.json configs[1], the paper's headline K20c workload): SGEMM,
100,000 independent pairs at n = 10 and at n = 16, N/N, general alpha and beta,
packed layout.  One step = one pass of the whole hot path over one batch of each
size (two library calls).  Two input sets (1.14 GB) alternate between steps, so
a step never finds its inputs in the 126 MB L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank owns its own 100,000-pair batches (weak scaling, no
data-path collective); the time is the max over ranks.  Prints ONE JSON line on
rank 0.  `value` is GFlop/s by the paper's convention (2n^3 per pair,
PAPER.md:567-570) over all ranks; GB/s and the roofline are reported beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: the paper's headline K20c workload (the default)
    "cfg2": dict(kind="s", sizes=(10, 16), batch=100_000, beta0=False, sets=2, scaling="weak",
                 text="cfg2: SGEMM 100,000 independent pairs at n=10 and at n=16, op N/N, general "
                      "alpha/beta, packed (minimal leading dimensions)",
                 l2="2 alternating input sets of 570 MB (> 126 MB L2)"),
    # configs[0]: small case (latency-bound; reported in us per step)
    "cfg1": dict(kind="s", sizes=(4,), batch=1_000, beta0=True, sets=1, scaling="weak",
                 text="cfg1: SGEMM 1,000 pairs of 4x4, N/N, alpha=1, beta=0",
                 l2="192 KB working set: L2-resident by construction (latency-bound case)"),
    # configs[4]: D/Z 16x16, 10^7 pairs sharded over the GPUs (strong scaling)
    "cfg5d": dict(kind="d", sizes=(16,), batch=10_000_000, beta0=False, sets=1, scaling="strong",
                  text="cfg5: DGEMM 16x16, 10^7 pairs in total split over the GPUs, general alpha/beta",
                  l2="inputs 61 GB >> 126 MB L2"),
    "cfg5z": dict(kind="z", sizes=(16,), batch=10_000_000, beta0=False, sets=1, scaling="strong",
                  text="cfg5: ZGEMM 16x16, 10^7 pairs in total split over the GPUs, general alpha/beta",
                  l2="inputs 123 GB >> 126 MB L2"),
}
KIND, SIZES, BATCH, GLOBAL_BATCH, BETA0, NSETS, SCALING = "s", (10, 16), 100_000, 100_000, False, 2, "weak"
RANGE = (0, 100_000)
WORKLOAD, L2NOTE = WORKLOADS["cfg2"]["text"], WORKLOADS["cfg2"]["l2"]
TYPENAME = {"s": "float", "d": "double", "c": "float2", "z": "double2"}
DTYPE = {"s": "f32", "d": "f64", "c": "c64 (f32 pairs)", "z": "c128 (f64 pairs)"}


def configure(name, world, rank):
    """Select the workload; per-rank pair range (weak: fixed per rank, strong: split)."""
    global KIND, SIZES, BATCH, GLOBAL_BATCH, BETA0, NSETS, SCALING, RANGE, WORKLOAD, L2NOTE
    from paper_1304_7053_b200 import shard

    w = WORKLOADS[name]
    KIND, SIZES, BETA0, NSETS, SCALING = w["kind"], w["sizes"], w["beta0"], w["sets"], w["scaling"]
    WORKLOAD, L2NOTE = w["text"], w["l2"]
    if SCALING == "weak":
        RANGE = shard.weak_range(w["batch"], rank)
        GLOBAL_BATCH = w["batch"] * world
    else:
        RANGE = shard.strong_range(w["batch"], world, rank)
        GLOBAL_BATCH = w["batch"]
    BATCH = RANGE[1] - RANGE[0]
METRIC = "batched GEMM GFlop/s and HBM GB/s (% of peak) vs size n=1..16, 1-8 B200"
PAPER_CONTEXT = {"hw": "Tesla K20c", "alpha1_beta0_gflops": {"10": 104, "16": 216},
                 "cite": "PAPER.md:37-38, 757, 763 (Table 1)"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get("bench_dominant_kernel", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0, t1):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = []
        for ts, line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((ts, float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        inside = [r for r in rows if t0 - 0.05 <= r[0] <= t1 + 0.05] or rows[-3:]
        if not inside:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inside for i, v in enumerate(r[3])
                          if v.lower() in ("active", "1", "yes")})
        return {"sm_mhz": statistics.median(r[1] for r in inside),
                "sm_max_mhz": max(r[2] for r in inside), "reasons": reasons,
                "samples": len(inside)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(args.dist_backend)
    return world, rank, local


def make_inputs(rank, set_id, device):
    """Seeded synthetic batch for one rank: its global pair range RANGE of the workload."""
    import txinputs
    from paper_1304_7053_b200 import shard

    out = {}
    for n in SIZES:
        key = lambda name: txinputs.stream_key(txinputs.DEFAULT_SEED, "bench", set_id, KIND, n, name)
        lo, hi = shard.element_range(RANGE, n * n)
        out[n] = tuple(txinputs.values_torch(KIND, key(nm), lo, hi - lo, device)
                       for nm in ("A", "B", "C"))
    return out


def scalars():
    import txinputs

    ka = txinputs.stream_key(txinputs.DEFAULT_SEED, "bench", "alpha")
    kb = txinputs.stream_key(txinputs.DEFAULT_SEED, "bench", "beta")
    if BETA0:
        return 1.0, 0.0
    return txinputs.scalar(KIND, ka), txinputs.scalar(KIND, kb)


def cpu_oracle_rate(seconds_budget=12.0, pairs=4000):
    """The oracle as it stands (single-threaded C loop), run by T host threads on
    contiguous sub-batches of a bounded sample of the workload; GFlop/s."""
    import numpy as np

    import oracle
    import txinputs
    from paper_1304_7053_b200 import model

    alpha, beta = scalars()
    T = len(os.sched_getaffinity(0))
    per = {}
    for n in SIZES:
        key = lambda name: txinputs.stream_key(txinputs.DEFAULT_SEED, "bench", 0, KIND, n, name)
        e = n * n
        per[n] = [txinputs.values_numpy(KIND, key(nm), 0, pairs * e).copy() for nm in ("A", "B", "C")]
    flops_one = sum(model.flops(KIND, n, n, n, pairs) for n in SIZES)

    def work(tid, reps, out):
        t = 0.0
        for _ in range(reps):
            for n in SIZES:
                A, B, C = per[n]
                Cw = C.copy()
                t0 = time.perf_counter()
                oracle.gemm_batched(KIND, "N", "N", n, n, n, alpha, A, n, n * n, B, n, n * n, beta,
                                    Cw, n, n * n, pairs)
                t += time.perf_counter() - t0
        out[tid] = t

    # calibrate on one thread, then size the multi-threaded run to the budget
    o = {}
    work(0, 1, o)
    t1 = max(o[0], 1e-6)
    reps = max(1, int(seconds_budget / t1 / 2))
    o = {}
    ths = [threading.Thread(target=work, args=(i, reps, o)) for i in range(T)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    wall = time.perf_counter() - t0
    total = flops_one * reps * T
    return {"value": round(total / wall / 1e9, 3), "unit": "GFlop/s", "cores": T, "kind": "oracle",
            "sample": f"{reps} x {pairs} pairs per size (n=10 and n=16) per thread on {T} "
                      f"threads, each thread running the unchanged single-threaded oracle",
            "single_thread_gflops": round(flops_one / t1 / 1e9, 3)}


def run_reference(args, world, rank):
    """--impl reference: the oracle, as it stands, on the host cores; each step a
    bounded sample of the workload."""
    if rank != 0:
        return
    import oracle  # noqa: F401
    from paper_1304_7053_b200 import model

    pairs = 2000
    T = len(os.sched_getaffinity(0))
    import numpy as np

    import txinputs

    alpha, beta = scalars()
    data = {}
    for n in SIZES:
        key = lambda name: txinputs.stream_key(txinputs.DEFAULT_SEED, "bench", 0, KIND, n, name)
        e = n * n
        data[n] = [txinputs.values_numpy(KIND, key(nm), 0, pairs * T * e).copy()
                   for nm in ("A", "B", "C")]

    def step():
        def w(t):
            for n in SIZES:
                A, B, C = data[n]
                e = n * n
                sl = slice(t * pairs * e, (t + 1) * pairs * e)
                oracle.gemm_batched(KIND, "N", "N", n, n, n, alpha, A[sl], n, e, B[sl], n, e, beta,
                                    C[sl].copy(), n, e, pairs)
        ths = [threading.Thread(target=w, args=(t,)) for t in range(T)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    flops = sum(model.flops(KIND, n, n, n, pairs * T) for n in SIZES) * args.steps
    byts = sum(model.bytes_moved(KIND, n, n, n, pairs * T, True, not BETA0) for n in SIZES) * args.steps
    val = flops / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GFlop/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": SCALING, "vs_baseline": None, "dtype": DTYPE[KIND], "data": "synthetic",
            "gbps": round(byts / dt / 1e9, 3),
            "config": {"workload": WORKLOAD, "kind": KIND, "sizes": list(SIZES), "batch": GLOBAL_BATCH,
                       "reference_sample": f"{pairs * T} pairs per size per step"},
            "cpu_baseline": {"value": round(val, 3), "unit": "GFlop/s", "cores": T,
                             "kind": "oracle",
                             "sample": f"{pairs} pairs per size per thread per step, {T} threads"},
            "e2e": {"value": round(val, 3), "unit": "GFlop/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def max_over_ranks(v, dev, args):
    import torch

    t = torch.tensor([v], device=dev if args.dist_backend == "nccl" else "cpu")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, world, rank, local):
    import torch

    import paper_1304_7053_b200 as tx
    from paper_1304_7053_b200 import model

    local = local % torch.cuda.device_count()  # several ranks per GPU only when testing (gloo)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tx.lib()  # fails loudly if the CUDA library is missing: no fallback
    alpha, beta = scalars()
    sets = [make_inputs(rank, s, dev) for s in range(NSETS)]
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    n_launch = [0]

    def call(n, A, B, C):
        rc = tx.tx_gemm_batched(KIND, "N", "N", n, n, n, alpha, A, n, n * n, B, n, n * n, beta, C,
                                n, n * n, BATCH, stream)
        if rc != 0:
            raise tx.TxError(rc, tx.status_string(rc))
        n_launch[0] += tx.last_path()[1]

    K, W = args.steps, args.warmup

    def step(i):
        s = sets[i % NSETS]
        for n in SIZES:
            call(n, *s[n])

    for i in range(W):
        step(i)
    n_launch[0] = 0
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.2)  # let the sampler attach before the timed region
    # ---- timed region: K steps, events only at the two ends, so consecutive
    # launches keep their programmatic-dependent-launch overlap
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.time()
    start.record(stream)
    for i in range(K):
        step(i)
    end.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    ms = start.elapsed_time(end)
    launches = n_launch[0]
    # ---- roofline of each kernel: R back-to-back launches of that size alone
    # (alternating input sets), CUDA events on the launch stream at both ends
    R = max(20, min(K, 200))
    per_launch = {}
    for n in SIZES:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(R):
            call(n, *sets[i % NSETS][n])
        b.record(stream)
        torch.cuda.synchronize()
        per_launch[n] = a.elapsed_time(b) / R
    # ---- per-launch events (each launch bracketed; breaks the launch overlap):
    # the kernel's share of the step, to compare with the ncu launch list
    evs = []
    for i in range(min(K, 50)):
        s_ = sets[i % NSETS]
        for n in SIZES:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            call(n, *s_[n])
            b.record(stream)
            evs.append((n, a, b))
    torch.cuda.synchronize()
    clocks = clk.stop(t_wall0, t_wall1)
    evented = {n: statistics.mean(a.elapsed_time(b) for m_, a, b in evs if m_ == n) for n in SIZES}
    if world > 1:
        ms = max_over_ranks(ms, dev, args)

    flops_step = sum(model.flops(KIND, n, n, n, BATCH) for n in SIZES)
    bytes_step = sum(model.bytes_moved(KIND, n, n, n, BATCH, True, not BETA0) for n in SIZES)
    value = flops_step * K * world / (ms / 1e3) / 1e9
    gbps = bytes_step * K * world / (ms / 1e3) / 1e9
    dom = max(SIZES)
    dom_bytes = model.bytes_moved(KIND, dom, dom, dom, BATCH, True, not BETA0)
    peak, peak_src = peaks()
    achieved = dom_bytes / (per_launch[dom] / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(),
                "kernel": f"bulk_kernel<{TYPENAME[KIND]},{dom},{dom},{dom},N,N,beta{'==' if BETA0 else '!='}0>",
                "algorithmic_bytes_per_launch": dom_bytes,
                "launch_ms": round(per_launch[dom], 5),
                "launch_ms_evented": round(evented[dom], 5),
                "share_of_step_evented": round(evented[dom] / sum(evented.values()), 4),
                "timing": f"{R} back-to-back launches, CUDA events at both ends",
                "peak_source": peak_src,
                "per_size_gbps": {str(n): round(model.bytes_moved(KIND, n, n, n, BATCH, True, not BETA0)
                                                / (per_launch[n] / 1e3) / 1e9, 1) for n in SIZES}}

    # ---- end to end through the host-buffer C-ABI entry (pinned host memory) ----
    e2e = None
    if not args.no_e2e:
        # end to end over at most 2*10^5 pairs of the rank's batch (pinned host memory)
        EB = min(BATCH, 200_000)
        host = {n: tuple(x[: EB * n * n].cpu().pin_memory() for x in sets[0][n]) for n in SIZES}
        staging = {n: tuple(torch.empty_like(x, device=dev) for x in host[n]) for n in SIZES}
        h2d = sum((x.numel() * x.element_size()) for n in SIZES for x in host[n])
        d2h = sum(host[n][2].numel() * host[n][2].element_size() for n in SIZES)

        def e2e_step():
            for n in SIZES:
                hA, hB, hC = host[n]
                dA, dB, dC = staging[n]
                rc = tx.tx_gemm_batched_hostio(KIND, "N", "N", n, n, n, alpha, hA, n, n * n, hB, n,
                                               n * n, beta, hC, n, n * n, EB, stream, dA, dB, dC)
                if rc != 0:
                    raise tx.TxError(rc, tx.status_string(rc))

        KE = max(1, min(K, 20))
        for _ in range(min(W, 3)):
            e2e_step()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(KE):
            e2e_step()
        s1.record(stream)
        torch.cuda.synchronize()
        ems = s0.elapsed_time(s1)
        if world > 1:
            ems = max_over_ranks(ems, dev, args)
        flops_e2e = sum(model.flops(KIND, n, n, n, EB) for n in SIZES)
        e2e = {"value": round(flops_e2e * KE * world / (ems / 1e3) / 1e9, 2), "unit": "GFlop/s",
               "pairs_per_size_per_step": EB,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": KE,
               "api": "tx_gemm_batched_hostio_s (host buffers, copies inside the timed region)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_rate()

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GFlop/s", "n_gpus": world,
                "steps": K, "warmup": W, "ms_per_step": round(ms / K, 5),
                "higher_is_better": True, "scaling": SCALING, "vs_baseline": None,
                "dtype": DTYPE[KIND],
                "data": "synthetic (seeded counter-based U[-1,1), txinputs)",
                "config": {"workload": WORKLOAD, "kind": KIND, "sizes": list(SIZES),
                           "batch_per_gpu": BATCH, "global_batch": GLOBAL_BATCH,
                           "parallelism": f"dp{world} (independent pairs, no collective)",
                           "l2": L2NOTE},
                "gbps": round(gbps, 1), "hbm_frac": round(gbps / peak, 4),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks, "paper_context": PAPER_CONTEXT}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS),
                    help="cfg2 (default, BASELINE configs[1]), cfg1 (configs[0]), cfg5d/cfg5z "
                         "(configs[4], 10^7 pairs split over the GPUs)")
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"),
                    help="process-group backend for the barrier / max-over-ranks (gloo: testing "
                         "several ranks on one GPU)")
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    configure(args.workload, world, rank)
    if args.impl == "reference":
        run_reference(args, world, rank)  # rank 0 only; other ranks exit 0
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
