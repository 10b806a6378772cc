"""Run one case a few times (for ncu): python tools/prof_case.py KIND N OPS BETA0 [BATCH]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1304_7053_b200 as tx  # noqa: E402
import txinputs  # noqa: E402

kind, n, ops, b0 = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4] == "1"
batch = int(sys.argv[5]) if len(sys.argv) > 5 else 1_000_000
A = txinputs.values_torch(kind, 1, 0, n * n * batch, "cuda")
B = txinputs.values_torch(kind, 2, 0, n * n * batch, "cuda")
C = txinputs.values_torch(kind, 3, 0, n * n * batch, "cuda")
for _ in range(4):
    rc = tx.tx_gemm_batched(kind, ops[0], ops[1], n, n, n, 0.5, A, n, n * n, B, n, n * n,
                            0 if b0 else 0.25, C, n, n * n, batch)
    assert rc == 0
torch.cuda.synchronize()
print("ok", tx.last_path())
