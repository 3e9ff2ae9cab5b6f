"""Sizes beyond 2^31 elements (positions and offsets above the signed 32-bit range,
the interface allows n < 2^32): a stable multisplit is checked through properties
that determine it uniquely at any size -- bucket ids non-decreasing, bucket offsets
equal to the bucket counts of the input, values (= input indices) a permutation,
increasing inside every bucket, and keys_out[i] = keys_in[values_out[i]]."""
import pytest
import torch

from gen import device as gdev
from gen import inputs as gen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ms = pytest.importorskip("paper_1701_01189_b200")

CH = 1 << 27


def u64(t):
    return t.to(torch.int64) & 0xFFFFFFFF


@pytest.mark.parametrize("m", [32, 256])
def test_pairs_beyond_2p31(m):
    n = (1 << 31) + 12345
    delta = -(-(1 << 32) // m)
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(k, 77 + m, kind=gen.DELTA, m=m, delta=delta, dist=gen.DIST_SKEW, alpha=0.5)
    v = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.values_(v, 1, parity=True)  # v_i = i
    ko, vo, off = ms.multisplit(k, v, bucket=ms.Delta(m))
    torch.cuda.synchronize()
    off = u64(off.cpu())
    assert int(off[0]) == 0 and int(off[m]) == n
    counts = torch.zeros(m, dtype=torch.int64, device="cuda")
    seen = torch.zeros(n, dtype=torch.uint8, device="cuda")
    prev_b, prev_v = -1, -1
    for s in range(0, n, CH):
        e = min(n, s + CH)
        kin = u64(k[s:e])
        counts += torch.bincount(torch.clamp(kin // delta, max=m - 1), minlength=m)
        ks, vs = u64(ko[s:e]), u64(vo[s:e])
        b = torch.clamp(ks // delta, max=m - 1)
        assert bool((b[1:] >= b[:-1]).all()) and int(b[0]) >= prev_b, "bucket ids must not decrease"
        same = b[1:] == b[:-1]
        assert bool((vs[1:][same] > vs[:-1][same]).all()), "stability inside a bucket"
        if int(b[0]) == prev_b:
            assert int(vs[0]) > prev_v
        assert bool((u64(k[vs]) == ks).all()), "keys_out[i] = keys_in[values_out[i]]"
        seen[vs] = 1
        # every output position lies inside the offsets of its bucket
        pos = torch.arange(s, e, device="cuda", dtype=torch.int64)
        offd = off.cuda()
        assert bool(((pos >= offd[b]) & (pos < offd[b + 1])).all())
        prev_b, prev_v = int(b[-1]), int(vs[-1])
    assert bool(seen.all()), "values_out is a permutation of the input indices"
    assert torch.equal(counts.cpu(), off[1:] - off[:-1])


def test_keys_beyond_2p31_m2():
    n = (1 << 31) + 777
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(k, 5)
    ko, _, off = ms.multisplit(k, None, bucket=ms.Delta(2))
    torch.cuda.synchronize()
    off = u64(off.cpu())
    ones = 0
    for s in range(0, n, CH):
        ones += int((u64(k[s:min(n, s + CH)]) >> 31).sum())
    assert int(off[1]) == n - ones and int(off[2]) == n
    # bucket 0 then bucket 1, each a stable copy: keys with the top bit clear come first, in order
    for s in range(0, n, CH):
        e = min(n, s + CH)
        b = u64(ko[s:e]) >> 31
        pos = torch.arange(s, e, device="cuda")
        assert bool((b == (pos >= int(off[1])).to(torch.int64)).all())
    lo = int(off[1])
    ref = k[(u64(k) >> 31) == 0]
    assert torch.equal(ko[:lo], ref)


def test_sort_pairs_beyond_2p31():
    """the 4 x 8-bit sort (configs[3]'s schedule) at 2^31 + 5 pairs"""
    n = (1 << 31) + 5
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(k, 9)
    v = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.values_(v, 1, parity=True)
    ko, vo = ms.radix_sort(k, v, bits_per_pass=8)
    torch.cuda.synchronize()
    seen = torch.zeros(n, dtype=torch.uint8, device="cuda")
    prev_k, prev_v = -1, -1
    for s in range(0, n, CH):
        e = min(n, s + CH)
        ks, vs = u64(ko[s:e]), u64(vo[s:e])
        assert bool((ks[1:] >= ks[:-1]).all()) and int(ks[0]) >= prev_k, "sorted"
        same = ks[1:] == ks[:-1]
        assert bool((vs[1:][same] > vs[:-1][same]).all()), "stable"
        if int(ks[0]) == prev_k:
            assert int(vs[0]) > prev_v
        assert bool((u64(k[vs]) == ks).all())
        seen[vs] = 1
        prev_k, prev_v = int(ks[-1]), int(vs[-1])
    assert bool(seen.all())


@pytest.mark.parametrize("n", [(1 << 30) - 1, 1 << 30])
@pytest.mark.parametrize("pairs", [False, True])
def test_sort_at_the_one_pass_limit(n, pairs):
    """The one-pass sort's look-back words hold 30-bit prefixes: n = 2^30 - 1 is its largest
    input, n = 2^30 takes the per-digit multisplit; both sort stably (checked on device)."""
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(k, 11 + n % 7)
    k[::3] &= 0xFF00FF  # duplicates: stability visible
    v = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.values_(v, 1, parity=True)  # v_i = i
    if pairs:
        ko, vo = ms.radix_sort(k, v, bits_per_pass=8)
    else:
        ko, _ = ms.radix_sort(k, None, bits_per_pass=8)
        vo = None
    torch.cuda.synchronize()
    seen = torch.zeros(n, dtype=torch.uint8, device="cuda") if pairs else None
    hist_in = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
    hist_out = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
    prev_k, prev_v = -1, -1
    for s in range(0, n, CH):
        e = min(n, s + CH)
        ks = u64(ko[s:e])
        assert bool((ks[1:] >= ks[:-1]).all()) and int(ks[0]) >= prev_k, "sorted"
        hist_in += torch.bincount(u64(k[s:e]) >> 16, minlength=1 << 16)
        hist_out += torch.bincount(ks >> 16, minlength=1 << 16)
        if pairs:
            vs = u64(vo[s:e])
            same = ks[1:] == ks[:-1]
            assert bool((vs[1:][same] > vs[:-1][same]).all()), "stable"
            if int(ks[0]) == prev_k:
                assert int(vs[0]) > prev_v
            assert bool((u64(k[vs]) == ks).all())
            seen[vs] = 1
            prev_v = int(vs[-1])
        prev_k = int(ks[-1])
    assert torch.equal(hist_in, hist_out), "the same multiset of keys"
    if pairs:
        assert bool(seen.all())
