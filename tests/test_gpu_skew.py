"""Skewed inputs through the m > 32 postscan, whose hot bucket (more than T/16 of
a tile) is ranked by ballots instead of increments: alpha-uniform keys
with 90 %, 70 % and 10 % hot shares, the hot bucket first / last / inside, two
hot buckets, and ragged tails, bit-exact against the oracle."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gen

pytestmark = pytest.mark.gpu
ms = pytest.importorskip("paper_1701_01189_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("m", [33, 64, 128, 256])
@pytest.mark.parametrize("hot_share", [0.9, 0.7, 0.1])
@pytest.mark.parametrize("hot", ["first", "last", "mid"])
@pytest.mark.parametrize("pairs", [False, True])
def test_hot_bucket(m, hot_share, hot, pairs):
    n = 5 * 16384 + 4321
    r = np.random.default_rng(m * 100 + int(hot_share * 10))
    keys = r.integers(0, m, n).astype(np.uint32)
    h = {"first": 0, "last": m - 1, "mid": m // 3}[hot]
    keys[r.random(n) < hot_share] = h
    vals = np.arange(n, dtype=np.uint32) if pairs else None
    ek, ev, eo = oracle.multisplit(keys, oracle.identity(m), vals)
    ko, vo, off = ms.multisplit(dev(keys), dev(vals) if pairs else None, bucket=ms.Identity(m))
    assert np.array_equal(host(off), eo) and np.array_equal(host(ko), ek)
    if pairs:
        assert np.array_equal(host(vo), ev)


@pytest.mark.parametrize("pairs", [False, True])
def test_two_hot_buckets_and_changing_hot(pairs):
    """tiles whose hot bucket changes from tile to tile, and two buckets of 45 % each"""
    m, n = 256, 9 * 16384 + 17
    r = np.random.default_rng(3)
    keys = r.integers(0, m, n).astype(np.uint32)
    tile = np.arange(n) // 4096
    sel = r.random(n) < 0.8
    keys[sel] = (tile[sel] * 37 % m).astype(np.uint32)  # a different hot bucket every 4096 keys
    keys2 = r.integers(0, m, n).astype(np.uint32)
    u = r.random(n)
    keys2[u < 0.45] = 7
    keys2[(u >= 0.45) & (u < 0.9)] = 8
    for k in (keys, keys2):
        vals = np.arange(n, dtype=np.uint32) if pairs else None
        ek, ev, eo = oracle.multisplit(k, oracle.identity(m), vals)
        ko, vo, off = ms.multisplit(dev(k), dev(vals) if pairs else None, bucket=ms.Identity(m))
        assert np.array_equal(host(off), eo) and np.array_equal(host(ko), ek)
        if pairs:
            assert np.array_equal(host(vo), ev)
