"""Pins for the oracle's splitter buckets (reading R27) and for m > 256
(Sec.6.3): each check ties orc_multisplit_ex / orc_bucket_ex to
something other than itself -- numpy's searchsorted and stable argsort, Eq.(1)
evaluated by brute force, the closed-form equivalence with delta buckets, and
the invariants of a stable multisplit."""
import numpy as np
import pytest

import oracle
from tests.test_oracle_pins import eq1_positions


def rng(seed):
    return np.random.default_rng(seed)


def random_splitters(r, m):
    return np.sort(r.choice(1 << 32, size=m - 1, replace=False).astype(np.uint64)).astype(np.uint32)


@pytest.mark.parametrize("m", [2, 3, 7, 32, 33, 255, 256, 257, 1000])
def test_splitter_bucket_is_upper_bound(m):
    # f(u) = j with s_j <= u < s_{j+1} = number of interior splitters <= u
    r = rng(m)
    spl = random_splitters(r, m)
    fn = oracle.splitters(spl)
    keys = np.concatenate([r.integers(0, 1 << 32, 2000, dtype=np.uint64).astype(np.uint32),
                           spl, spl - 1, spl + 1, np.array([0, 0xFFFFFFFF], np.uint32)])
    got = np.array([oracle.bucket_of(fn, int(k)) for k in keys])
    assert np.array_equal(got, np.searchsorted(spl, keys, side="right"))


def test_splitter_edges_by_hand():
    # splitters {10, 20}: [0,10) -> 0, [10,20) -> 1, [20, 2^32) -> 2
    fn = oracle.splitters([10, 20])
    for u, b in [(0, 0), (9, 0), (10, 1), (19, 1), (20, 2), (0xFFFFFFFF, 2)]:
        assert oracle.bucket_of(fn, u) == b
    ko, _, off = oracle.multisplit(np.array([25, 3, 10, 19, 0, 20], np.uint32), fn)
    assert ko.tolist() == [3, 0, 10, 19, 25, 20] and off.tolist() == [0, 2, 4, 6]


@pytest.mark.parametrize("m", [2, 5, 64, 256, 300, 4096, 65536])
def test_splitter_multisplit_is_stable_argsort(m):
    r = rng(100 + m)
    spl = random_splitters(r, m)
    n = 20000
    keys = r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, off = oracle.multisplit(keys, oracle.splitters(spl), vals)
    b = np.searchsorted(spl, keys, side="right")
    order = np.argsort(b, kind="stable")
    assert np.array_equal(ko, keys[order]) and np.array_equal(vo, vals[order])
    assert np.array_equal(off, np.concatenate([[0], np.cumsum(np.bincount(b, minlength=m))]).astype(np.uint32))


@pytest.mark.parametrize("m", [3, 17, 256, 300])
def test_splitters_equal_delta_buckets(m):
    # closed form: splitters at j*D (j = 1..m-1) are exactly delta buckets of width D
    # whenever (m-1)*D < 2^32
    d = (1 << 32) // m
    spl = np.arange(1, m, dtype=np.uint64) * d
    keys = rng(m).integers(0, 1 << 32, 5000, dtype=np.uint64).astype(np.uint32)
    a = oracle.multisplit(keys, oracle.splitters(spl.astype(np.uint32)))
    b = oracle.multisplit(keys, oracle.delta(m, d))
    assert all(np.array_equal(x, y) for x, y in zip(a, b) if x is not None)


def test_splitters_m1_is_copy_and_invalid_rejected():
    keys = np.array([7, 3, 3, 1], np.uint32)
    ko, _, off = oracle.multisplit(keys, oracle.splitters([]))
    assert np.array_equal(ko, keys) and off.tolist() == [0, 4]
    for bad in ([5, 5], [9, 4], [1, 2, 2]):
        with pytest.raises(oracle.OracleError):
            oracle.multisplit(keys, oracle.splitters(bad))


@pytest.mark.parametrize("kind", ["delta", "identity", "splitters", "radix"])
def test_large_m_brute_force_eq1(kind):
    # Eq.(1) literally, O(n^2), at m beyond the paper's 256
    r = rng(7)
    m, n = 1000, 1500
    if kind == "delta":
        fn = oracle.delta(m)
        keys = r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    elif kind == "identity":
        fn = oracle.identity(m)
        keys = r.integers(0, m, n).astype(np.uint32)
    elif kind == "radix":
        fn = oracle.radix(4, 10)
        m = fn.m
        keys = r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    else:
        fn = oracle.splitters(random_splitters(r, m))
        keys = r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, off = oracle.multisplit(keys, fn, vals)
    b = np.array([oracle.bucket_of(fn, int(k)) for k in keys])
    p = eq1_positions(b)
    exp = np.empty(n, np.uint32)
    exp[p] = keys
    assert np.array_equal(ko, exp)
    assert np.array_equal(off[1:] - off[:-1], np.bincount(b, minlength=m))
    # invariants: permutation, non-decreasing buckets, stability
    assert np.array_equal(np.sort(ko), np.sort(keys))
    bo = np.array([oracle.bucket_of(fn, int(k)) for k in ko])
    assert np.all(np.diff(bo) >= 0)
    same = bo[1:] == bo[:-1]
    assert np.all(vo[1:][same] > vo[:-1][same])


def test_large_m_delta_closed_form():
    # m = 2^16 delta buckets with the default width 2^16: f(u) = u >> 16, so the multisplit
    # equals a stable sort by the top 16 bits (numpy stable argsort)
    r = rng(9)
    keys = r.integers(0, 1 << 32, 100000, dtype=np.uint64).astype(np.uint32)
    ko, _, off = oracle.multisplit(keys, oracle.delta(65536))
    assert np.array_equal(ko, keys[np.argsort(keys >> 16, kind="stable")])
    assert off[-1] == keys.size


def test_large_m_limits():
    keys = np.array([1, 2], np.uint32)
    with pytest.raises(oracle.OracleError):
        oracle.multisplit(keys, oracle.delta(65537))
    with pytest.raises(oracle.OracleError):
        oracle.multisplit(keys, oracle.radix(0, 17))
