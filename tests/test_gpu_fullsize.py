"""Full-size parity at BASELINE.json's configurations, in the launch
configuration bench.py times (same entry points, same tile size, device-side
input generation).  Multisplit results are compared with the C oracle element
by element; the 2^28 radix sort is checked through properties that determine
the stable sort uniquely (sorted keys + values = input index permutation,
increasing inside equal keys) plus sampled elements against the oracle."""
import numpy as np
import pytest
import torch

import oracle
from gen import device as gdev
from gen import inputs as gen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ms = pytest.importorskip("paper_1701_01189_b200")


def host(t):
    return t.cpu().numpy().view(np.uint32)


def gen_dev(n, seed, parity_vals=True, **gk):
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(k, seed, **gk)
    v = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.values_(v, seed, parity=parity_vals)
    return k, v


@pytest.mark.parametrize("m", [2, 8, 32])
def test_c2_keys_and_pairs_2p25(m):
    n = 1 << 25
    ob = oracle.delta(m)
    k, v = gen_dev(n, 0x5EED, kind=gen.DELTA, m=m, delta=ob.delta)
    kh, vh = host(k), host(v)
    ek, ev, eo = oracle.multisplit(kh, ob, vh)
    ko, _, off = ms.multisplit(k, None, bucket=ms.Delta(m))
    assert np.array_equal(host(ko), ek) and np.array_equal(host(off), eo)
    ko, vo, off = ms.multisplit(k, v, bucket=ms.Delta(m))
    assert np.array_equal(host(ko), ek) and np.array_equal(host(vo), ev)


@pytest.mark.parametrize("m", [64, 256])
@pytest.mark.parametrize("kind", ["identity", "radix"])
@pytest.mark.parametrize("dist", [gen.DIST_UNIFORM, gen.DIST_SKEW])
def test_c3_pairs_2p27(m, kind, dist):
    n = 1 << 27
    bits = m.bit_length() - 1
    if kind == "identity":
        ob, pb, gk = oracle.identity(m), ms.Identity(m), dict(kind=gen.IDENTITY, m=m)
    else:
        ob, pb, gk = oracle.radix(0, bits), ms.Radix(0, bits), dict(kind=gen.RADIX, m=m, shift=0, bits=bits)
    k, v = gen_dev(n, 0x5EED + m, dist=dist, alpha=0.1, **gk)
    kh, vh = host(k), host(v)
    ek, ev, eo = oracle.multisplit(kh, ob, vh)
    ko, vo, off = ms.multisplit(k, v, bucket=pb)
    assert np.array_equal(host(ko), ek) and np.array_equal(host(vo), ev) and np.array_equal(host(off), eo)


@pytest.mark.parametrize("r", [8, 5])
def test_c4_radix_sort_pairs_2p28(r):
    """configs[3] as benched (r = 8: 4 x 8-bit passes over [0, 32), also the library default) and 5-bit digits."""
    n = 1 << 28
    k, v = gen_dev(n, 0x5EED)
    ko, vo = ms.radix_sort(k, v, begin_bit=0, end_bit=32, bits_per_pass=r)
    kh = host(k)
    ok, ov = host(ko), host(vo)
    assert np.all(ok[1:] >= ok[:-1])                       # sorted
    assert np.array_equal(kh[ov], ok)                      # values are the input indices of the keys
    same = ok[1:] == ok[:-1]
    assert np.all(ov[1:][same] > ov[:-1][same])            # stable
    assert np.unique(ov).size == n                         # a permutation
    # sampled elements against the oracle on a bounded prefix-free sample:
    # the rank of key x in the sorted output = number of keys < x (Eq.1 for identity digits)
    rng = np.random.default_rng(1)
    ks = np.sort(kh)
    for i in rng.integers(0, n, 64):
        assert ok[i] == ks[i]
    del ks
    ko2, _ = ms.radix_sort(k, bits_per_pass=r)
    assert torch.equal(ko2, ko)
    small_k, small_v = oracle.radix_sort(kh[:1 << 20], np.arange(1 << 20, dtype=np.uint32))
    ko3, vo3 = ms.radix_sort(k[:1 << 20].clone(), v[:1 << 20].clone(), bits_per_pass=r)
    assert np.array_equal(host(ko3), small_k) and np.array_equal(host(vo3), small_v)
