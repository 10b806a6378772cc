"""Run one strided (packed) case a few times (for ncu):
python tools/prof_ns_case.py KIND M N K OPS BETA0 [BATCH]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1304_7053_b200 as tx  # noqa: E402
import txinputs  # noqa: E402

kind, m, n, k, ops, b0 = sys.argv[1], *map(int, sys.argv[2:5]), sys.argv[5], sys.argv[6] == "1"
batch = int(sys.argv[7]) if len(sys.argv) > 7 else 1_000_000
A = txinputs.values_torch(kind, 1, 0, m * k * batch, "cuda")
B = txinputs.values_torch(kind, 2, 0, k * n * batch, "cuda")
C = txinputs.values_torch(kind, 3, 0, m * n * batch, "cuda")
lda = m if ops[0] == "N" else k
ldb = k if ops[1] == "N" else n
for _ in range(4):
    rc = tx.tx_gemm_batched(kind, ops[0], ops[1], m, n, k, 0.5, A, lda, m * k, B, ldb, k * n,
                            0 if b0 else 0.25, C, m, m * n, batch)
    assert rc == 0
torch.cuda.synchronize()
print("ok", tx.last_path())
