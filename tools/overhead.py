"""Per-launch fixed cost: time vs batch for back-to-back stream launches and for a
CUDA-graph replay of the same launches (s16 / s10, general alpha/beta)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1304_7053_b200 as tx  # noqa: E402
import txinputs  # noqa: E402


def bufs(n, batch, r):
    key = lambda nm: txinputs.stream_key(3, "ovh", n, r, nm)
    return [txinputs.values_torch("s", key(nm), 0, n * n * batch, "cuda") for nm in "ABC"]


def main():
    s = torch.cuda.Stream()
    for n in (16, 10):
        for batch in (10_000, 30_000, 100_000, 300_000, 1_000_000):
            R = 4
            sets = [bufs(n, batch, r) for r in range(R)]

            def call(i):
                A, B, C = sets[i % R]
                assert tx.tx_gemm_batched("s", "N", "N", n, n, n, 0.7, A, n, n * n, B, n, n * n, 0.3,
                                          C, n, n * n, batch, s) == 0
            reps = 40
            with torch.cuda.stream(s):
                for i in range(8):
                    call(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for i in range(reps):
                call(i)
            e1.record(s)
            torch.cuda.synchronize()
            t_stream = e0.elapsed_time(e1) / reps * 1e3
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for i in range(reps):
                    call(i)
            with torch.cuda.stream(s):
                g.replay()
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                e0.record(s)
                g.replay()
                e1.record(s)
            torch.cuda.synchronize()
            t_graph = e0.elapsed_time(e1) / reps * 1e3
            byts = 4 * 4 * n * n * batch
            print(json.dumps({"n": n, "batch": batch, "us_stream": round(t_stream, 2),
                              "us_graph": round(t_graph, 2),
                              "gbps_stream": round(byts / t_stream / 1e3, 1),
                              "gbps_graph": round(byts / t_graph / 1e3, 1)}), flush=True)
            del sets
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
