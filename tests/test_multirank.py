"""N > 1 path on CPU: two ranks (gloo, world size 2) each take their shard of
the batch, generate it from the global streams and compute it (here with the
oracle, since there is no GPU); the union must equal the unsharded batch
bitwise, and the max-over-ranks reduction of timings must be the max."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import txinputs
from paper_1304_7053_b200 import shard

KIND, N, PER_RANK = "d", 6, 37


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_result(lo, hi, mode):
    e = N * N
    key = lambda nm: txinputs.stream_key(5, "mr", nm)
    A = txinputs.values_numpy(KIND, key("A"), lo * e, (hi - lo) * e).copy()
    B = txinputs.values_numpy(KIND, key("B"), lo * e, (hi - lo) * e).copy()
    C = txinputs.values_numpy(KIND, key("C"), lo * e, (hi - lo) * e).copy()
    assert oracle.gemm_batched(KIND, "N", "T", N, N, N, 0.75, A, N, e, B, N, e, -0.5, C, N, e,
                               hi - lo) == 0
    return C


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if mode == "weak":
        lo, hi = shard.weak_range(PER_RANK, rank)
    else:
        lo, hi = shard.strong_range(PER_RANK * world + 1, world, rank)
    C = _shard_result(lo, hi, mode)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, C))
    t = torch.tensor([1.5 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((parts, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_two_ranks_union_equals_unsharded(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.5
    parts.sort(key=lambda t: t[0])
    lo0, hi_last = parts[0][0], parts[-1][1]
    # contiguous, disjoint cover
    for (a, b, _), (c, d, _) in zip(parts, parts[1:]):
        assert b == c
    full = _shard_result(lo0, hi_last, mode)
    got = np.concatenate([c for _, _, c in parts])
    assert np.array_equal(got.view(np.uint8), full.view(np.uint8))


def test_strong_range_spec_example():
    # N=10, 3 chunks -> [0,4), [4,7), [7,10)
    assert [shard.strong_range(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert shard.weak_range(100, 3) == (300, 400)
