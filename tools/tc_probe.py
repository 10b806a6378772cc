"""What tcgen05.mma kind::tf32 computes on the B200 (measurement tool, needs a GPU).

  python tools/tc_probe.py      (builds tools/libtcprobe.so from tools/tc_probe.cu)

Checks (JSON on stdout):
  layout    -- integer operands (exact in tf32): D == A B^T bit for bit, for the
               shared-memory layout / descriptors the 3xTF32 kernel uses;
  convert   -- B = I: D = tf32(A); which rounding the tensor core applies to fp32 inputs;
  accum     -- sums of exact tf32 products: D vs the exact sum rounded RN / RZ;
  split3    -- the 3xTF32 split (hi = rna(x), lo = rna(x - hi)), random U[-1,1) at K = 64:
               max |D - AB^T| / (|A||B|^T), fp64 reference.
"""
import ctypes
import json
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tools", "libtcprobe.so")


def tf32(x, mode):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    if mode == "rz":
        r = b & ~np.uint64(0x1FFF)
    elif mode == "rna":
        r = (b + np.uint64(0x1000)) & ~np.uint64(0x1FFF)
    else:  # rne
        lsb = (b >> np.uint64(13)) & np.uint64(1)
        r = (b + np.uint64(0xFFF) + lsb) & ~np.uint64(0x1FFF)
    return r.astype(np.uint32).view(np.float32)


def main():
    src = os.path.join(ROOT, "tools", "tc_probe.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SO, src])
    import torch

    L = ctypes.CDLL(SO)
    rng = np.random.default_rng(7)

    def run(A0, B0, N, K, A1=None, B1=None, nsets=1, M=128):
        A1 = np.zeros_like(A0) if A1 is None else A1
        B1 = np.zeros_like(B0) if B1 is None else B1
        t = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda() for x in (A0, A1, B0, B1)]
        D = torch.zeros(128, N, dtype=torch.float32, device="cuda")
        rc = L.tc_probe(*(ctypes.c_void_p(x.data_ptr()) for x in t), ctypes.c_void_p(D.data_ptr()),
                        N, K, nsets, M)
        assert rc == 0, rc
        return D.cpu().numpy()

    out = {}
    lay = []
    for N, K in ((32, 32), (64, 64), (16, 32), (48, 96), (256, 32)):
        A = rng.integers(-8, 9, (128, K)).astype(np.float32)
        B = rng.integers(-8, 9, (N, K)).astype(np.float32)
        D = run(A, B, N, K)
        ref = A.astype(np.float64) @ B.astype(np.float64).T
        lay.append({"N": N, "K": K, "exact": bool(np.array_equal(D, ref)),
                    "mismatch": int(np.sum(D != ref))})
    out["layout"] = lay

    A = (rng.standard_normal((128, 32)) * 2.0 ** rng.integers(-8, 8, (128, 32))).astype(np.float32)
    D = run(A, np.eye(32, dtype=np.float32), 32, 32)
    out["convert"] = {m: int(np.sum(D == tf32(A, m))) for m in ("rz", "rne", "rna")}
    out["convert"]["n"] = int(A.size)

    # accumulation: products exact (tf32 values with few bits), sums need rounding
    K = 32
    A = tf32((rng.standard_normal((128, K)) * 2.0 ** rng.integers(-12, 12, (128, K))).astype(np.float32), "rz")
    B = tf32(rng.standard_normal((32, K)).astype(np.float32), "rz")
    D = run(A, B, 32, K)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    rn = exact.astype(np.float32)
    rz = np.where(np.abs(rn.astype(np.float64)) > np.abs(exact),
                  np.nextafter(rn, np.float32(0)), rn)
    den = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)).T
    out["accum"] = {"eq_rn_of_exact": int(np.sum(D == rn)), "eq_rz_of_exact": int(np.sum(D == rz)),
                    "n": int(D.size),
                    "max_err_over_sumabs": float(np.max(np.abs(D - exact) / den)),
                    "max_err_ulps_of_result": float(np.max(np.abs(D - exact) /
                                                           np.maximum(np.abs(exact), 1e-30)) / 2 ** -23)}

    res = []
    for K in (32, 64, 128):
        A = rng.uniform(-1, 1, (128, K)).astype(np.float32)
        B = rng.uniform(-1, 1, (64, K)).astype(np.float32)
        Ah = tf32(A, "rna")
        Al = tf32((A - Ah).astype(np.float32), "rna")
        Bh = tf32(B, "rna")
        Bl = tf32((B - Bh).astype(np.float32), "rna")
        D3 = run(Ah, Bh, 64, K, Al, Bl, nsets=3)
        D1 = run(A, B, 64, K)
        ref = A.astype(np.float64) @ B.astype(np.float64).T
        den = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)).T
        res.append({"K": K, "max_err_3xtf32": float(np.max(np.abs(D3 - ref) / den)),
                    "max_err_1xtf32": float(np.max(np.abs(D1 - ref) / den))})
    out["split3"] = res

    # M = 64: A row i = (i + 1, 0, ...), B = e_0 -> D[i][j] = i + 1 for i < 64; where is row i?
    A = np.zeros((128, 32), np.float32)
    A[:64, 0] = np.arange(1, 65)
    A[64:, 0] = 1000 + np.arange(64)  # rows the M = 64 MMA must not read
    B = np.zeros((16, 32), np.float32)
    B[:, 0] = 1
    D = run(A, B, 16, 32, M=64)
    lanes = {}
    for ln in range(128):
        v = D[ln, 0]
        lanes[ln] = int(v) - 1 if 0 < v <= 64 and np.all(D[ln] == v) else None
    out["m64_row_of_lane"] = lanes
    rows = {r: [ln for ln, rr in lanes.items() if rr == r] for r in range(64)}
    out["m64_lane_of_row_rule_16x4"] = all(rows[r] == [32 * (r // 16) + r % 16] for r in range(64))
    # layout check at M = 64 with integers
    A = rng.integers(-8, 9, (128, 64)).astype(np.float32)
    B = rng.integers(-8, 9, (40, 64)).astype(np.float32)
    D = run(A, B, 40, 64, M=64)
    ref = A[:64].astype(np.float64) @ B.astype(np.float64).T
    got = np.stack([D[32 * (r // 16) + r % 16] for r in range(64)])
    out["m64_exact_16x4_rule"] = bool(np.array_equal(got, ref))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
