"""The seeded input generator (txinputs): numpy and torch paths agree bitwise,
shards equal slices of the unsharded stream, distributions are as stated."""
import numpy as np
import pytest

import txinputs as T


@pytest.mark.parametrize("kind", "sdcz")
@pytest.mark.parametrize("dist", ["uniform", "int"])
def test_numpy_equals_torch_cpu(kind, dist):
    k = T.stream_key(5, "x", kind)
    a = T.values_numpy(kind, k, 17, 3001, dist)
    b = T.values_torch(kind, k, 17, 3001, "cpu", dist, chunk=1000).numpy()
    assert a.dtype == b.dtype
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_shard_equals_slice():
    k = T.stream_key(1, "shard")
    full = T.values_numpy("z", k, 0, 1000)
    parts = [T.values_numpy("z", k, lo, hi - lo) for lo, hi in T.chunk_ranges(1000, 7)]
    assert np.array_equal(np.concatenate(parts), full)


def test_uniform_range_and_grid():
    x = T.values_numpy("d", T.stream_key(2, "u"), 0, 200000)
    assert x.min() >= -1 and x.max() < 1 and abs(x.mean()) < 0.01
    assert np.all((x + 1) * 2**52 == np.round((x + 1) * 2**52))
    y = T.values_numpy("s", T.stream_key(2, "u"), 0, 200000)
    assert np.all((y.astype(np.float64) + 1) * 2**23 == np.round((y.astype(np.float64) + 1) * 2**23))


def test_int_dist():
    x = T.values_numpy("c", T.stream_key(3, "i"), 0, 10000, "int")
    r = np.concatenate([x.real, x.imag])
    assert set(np.unique(r)) == set(range(-4, 5))


def test_scalar_rejection():
    for i in range(50):
        a = T.scalar("z", T.stream_key(4, "ab"), i)
        for c in (a.real, a.imag):
            assert 0.1 <= abs(c) < 1 and c not in (0.0, 1.0, -1.0)


@pytest.mark.parametrize("n,parts,want", [(10, 3, [(0, 4), (4, 7), (7, 10)]),
                                          (5, 2000, [(i, i + 1) for i in range(5)]),
                                          (0, 4, [])])
def test_chunk_ranges_spec_examples(n, parts, want):
    """SPEC.md:345-347."""
    assert T.chunk_ranges(n, parts) == want
