"""GPU parity of splitter buckets (reading R27) and of the m > 256 path
(Sec.6.3) against the oracle, element by element (bit-exact)."""
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


def spl_random(r, m):
    return np.sort(r.choice(1 << 32, size=m - 1, replace=False).astype(np.uint64)).astype(np.uint32)


def check(keys, vals, ob, pb):
    ek, ev, eo = oracle.multisplit(keys, ob, vals)
    ko, vo, off = ms.multisplit(dev(keys), None if vals is None else dev(vals), bucket=pb)
    assert np.array_equal(host(off), eo), "bucket offsets differ"
    assert np.array_equal(host(ko), ek), "keys differ"
    if vals is not None:
        assert np.array_equal(host(vo), ev), "values differ"
    assert ms.device_status() == 0


@pytest.mark.parametrize("m", [1, 2, 3, 8, 32, 33, 64, 255, 256])
@pytest.mark.parametrize("n", [0, 1, 1000, 8193, 1 << 20])
@pytest.mark.parametrize("pairs", [False, True])
def test_splitters_grid(m, n, pairs):
    r = np.random.default_rng(m * 7 + n)
    spl = spl_random(r, m)
    keys = gen.keys(n, seed=m + n)
    # a share of the keys sits exactly on, and next to, the splitters
    if n and m > 1:
        k = min(n // 4, 3 * (m - 1))
        pick = r.integers(0, m - 1, k)
        edge = spl[pick].astype(np.int64) + r.integers(-1, 2, k)
        keys[r.choice(n, k, replace=False)] = np.clip(edge, 0, 0xFFFFFFFF).astype(np.uint32)
    vals = gen.values(n, seed=1) if pairs else None
    check(keys, vals, oracle.splitters(spl), ms.Splitters(dev(spl)))


@pytest.mark.parametrize("m", [4, 32, 100, 256])
def test_splitters_quantiles_and_skew(m):
    """equal-count buckets (splitters at key quantiles, the sample-sort use) and a
    90 % hot bucket (alpha-uniform) at tile-spanning sizes"""
    n = 3 * 8192 * 4 + 77
    keys = gen.keys(n, seed=m)
    spl = np.unique(np.quantile(keys, np.linspace(0, 1, m + 1)[1:-1]).astype(np.uint32))
    if spl.size == m - 1:
        check(keys, gen.values(n, seed=2), oracle.splitters(spl), ms.Splitters(dev(spl)))
    r = np.random.default_rng(m)
    spl = spl_random(r, m)
    hot = keys.copy()
    sel = r.random(n) < 0.9
    hot[sel] = spl[m // 2 - 1] if m > 1 else 0
    check(hot, None, oracle.splitters(spl), ms.Splitters(dev(spl)))
    check(hot, gen.values(n, seed=3), oracle.splitters(spl), ms.Splitters(dev(spl)))


def test_splitters_equal_delta_on_gpu():
    # splitters at multiples of D reproduce the delta buckets of the same width
    m, n = 200, 1 << 18
    d = (1 << 32) // m
    spl = (np.arange(1, m, dtype=np.uint64) * d).astype(np.uint32)
    keys = gen.keys(n, seed=9)
    a = ms.multisplit(dev(keys), bucket=ms.Splitters(dev(spl)))
    b = ms.multisplit(dev(keys), bucket=ms.Delta(m, d))
    assert torch.equal(a[0], b[0]) and torch.equal(a[2], b[2])


def test_splitters_full_size_c2():
    """BASELINE configs[1] size (2^25 keys) with m = 32 and m = 256 splitter buckets"""
    n = 1 << 25
    keys = gen.keys(n, seed=0x5EED)
    for m in (32, 256):
        spl = spl_random(np.random.default_rng(m), m)
        check(keys, None, oracle.splitters(spl), ms.Splitters(dev(spl)))


# --------------------------------------------------------------------------- m > 256
def large_bucket(kind, m, r):
    if kind == "delta":
        return oracle.delta(m), ms.Delta(m), None
    if kind == "identity":
        return oracle.identity(m), ms.Identity(m), None
    if kind == "radix":
        bits = (m - 1).bit_length()
        return oracle.radix(3, bits), ms.Radix(3, bits), None
    spl = spl_random(r, m)
    t = dev(spl)
    return oracle.splitters(spl), ms.Splitters(t), t


@pytest.mark.parametrize("kind", ["delta", "identity", "radix", "splitters"])
@pytest.mark.parametrize("m", [257, 1000, 4096, 65536])
@pytest.mark.parametrize("n", [1, 1000, (1 << 20) + 3])
@pytest.mark.parametrize("pairs", [False, True])
def test_large_m(kind, m, n, pairs):
    r = np.random.default_rng(m + n)
    if kind == "radix":
        m = 1 << (m - 1).bit_length()
    ob, pb, _keep = large_bucket(kind, m, r)
    keys = r.integers(0, m, n).astype(np.uint32) if kind == "identity" else gen.keys(n, seed=n)
    check(keys, gen.values(n, seed=4) if pairs else None, ob, pb)


def test_large_m_skew_and_empty():
    n = 300000
    r = np.random.default_rng(1)
    keys = r.integers(0, 5000, n).astype(np.uint32)
    keys[r.random(n) < 0.9] = 4321
    check(keys, gen.values(n, seed=5), oracle.identity(5000), ms.Identity(5000))
    check(np.zeros(0, np.uint32), None, oracle.identity(5000), ms.Identity(5000))


def test_large_m_identity_domain_error():
    keys = np.array([1, 2, 70000, 3], np.uint32)
    ms.multisplit(dev(keys), bucket=ms.Identity(1000))
    assert ms.device_status() == 5  # MS_ERR_KEY_DOMAIN


def test_large_m_limits():
    with pytest.raises(ms.MultisplitError):
        ms.multisplit(dev(np.arange(10, dtype=np.uint32)), bucket=ms.Identity(65537))


@pytest.mark.parametrize("layout", ["clustered", "half", "cell_edges", "top_cell", "pairs_per_cell"])
@pytest.mark.parametrize("m", [32, 256])
@pytest.mark.parametrize("pairs", [False, True])
def test_splitter_cell_table(layout, m, pairs):
    """The staged cell table over the key's top bits (1024 cells for m <= 256
    kernels, 128 for the m <= 32 ones): crowded cells take the search, cell
    boundaries and the last cell are exact, cells with two splitters compare twice."""
    r = np.random.default_rng(m + len(layout))
    if layout == "clustered":    # every splitter in one cell: the fallback search
        spl = np.sort(r.choice(1 << 20, size=m - 1, replace=False).astype(np.uint32) + np.uint32(5 << 22))
    elif layout == "half":       # half crowded, half spread
        a = r.choice(1 << 18, size=(m - 1) // 2, replace=False).astype(np.uint64) + (7 << 22)
        b = r.choice(1 << 32, size=m - 1 - a.size, replace=False).astype(np.uint64)
        spl = np.unique(np.concatenate([a, b])).astype(np.uint32)
    elif layout == "cell_edges":  # splitters exactly on cell starts (2^22 and 2^25 multiples) and one below
        c = np.sort(r.choice(1024, size=(m - 1) // 2, replace=False)).astype(np.uint64)
        spl = np.unique(np.concatenate([c << 22, (c << 22) + 1, [(1 << 32) - 1]])).astype(np.uint32)
    elif layout == "top_cell":   # splitters near the top of the key domain
        spl = np.sort((np.uint64(1 << 32) - 1 - r.choice(1 << 21, size=m - 1, replace=False).astype(np.uint64))
                      .astype(np.uint32))
    else:                        # exactly two splitters per cell in some cells
        c = np.sort(r.choice(1024, size=(m - 1) // 2, replace=False)).astype(np.uint64)
        spl = np.unique(np.concatenate([(c << 22) + 100, (c << 22) + 200])).astype(np.uint32)
    spl = spl[: m - 1]
    mm = spl.size + 1
    n = 5 * 8192 + 333
    keys = gen.keys(n, seed=mm)
    k = n // 3  # a third of the keys on, just below and just above the splitters
    pick = r.integers(0, spl.size, k)
    edge = spl[pick].astype(np.int64) + r.integers(-1, 2, k)
    keys[r.choice(n, k, replace=False)] = np.clip(edge, 0, 0xFFFFFFFF).astype(np.uint32)
    vals = gen.values(n, seed=2) if pairs else None
    check(keys, vals, oracle.splitters(spl), ms.Splitters(dev(spl)))
