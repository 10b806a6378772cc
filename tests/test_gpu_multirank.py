"""The N > 1 data path on one GPU: two ranks (gloo process group, world size 2,
both on cuda:0) each run the LIBRARY on their shard of the batch, generated on
the device from the global counter-based streams (the pairs are
independent, so the path shards with no exchange).  The union of
the shards must equal the unsharded library call bitwise, and the max-over-ranks
reduction bench.py uses must return the max."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KIND, N = "z", 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _compute(lo, hi, ta="C", tb="N"):
    """Library call over global pairs [lo, hi) (inputs from the global streams)."""
    import torch

    import paper_1304_7053_b200 as tx
    import txinputs

    e = N * N
    key = lambda nm: txinputs.stream_key(5, "gpumr", KIND, nm)
    A = txinputs.values_torch(KIND, key("A"), lo * e, (hi - lo) * e, "cuda")
    B = txinputs.values_torch(KIND, key("B"), lo * e, (hi - lo) * e, "cuda")
    C = txinputs.values_torch(KIND, key("C"), lo * e, (hi - lo) * e, "cuda")
    alpha = txinputs.scalar(KIND, key("alpha"))
    beta = txinputs.scalar(KIND, key("beta"))
    rc = tx.tx_gemm_batched(KIND, ta, tb, N, N, N, alpha, A, N, e, B, N, e, beta, C, N, e, hi - lo)
    assert rc == 0, tx.status_string(rc)
    torch.cuda.synchronize()
    return C.cpu().numpy()


def _worker(rank, world, port, mode, total, q):
    import torch
    import torch.distributed as dist

    from paper_1304_7053_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    lo, hi = (shard.weak_range(total, rank) if mode == "weak"
              else shard.strong_range(total, world, rank))
    C = _compute(lo, hi)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, C))
    t = torch.tensor([1.5 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((parts, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_two_ranks_library_union_equals_unsharded(mode):
    import torch.multiprocessing as mp

    world, total = 2, 20_011  # strong: odd total, ranks get 10,006 and 10,005 pairs
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax == 2.5
    parts.sort(key=lambda t: t[0])
    for (a, b, _), (c, d, _) in zip(parts, parts[1:]):
        assert b == c
    full = _compute(parts[0][0], parts[-1][1])
    got = np.concatenate([c for _, _, c in parts])
    assert np.array_equal(got.view(np.uint8), full.view(np.uint8))
