"""Repeated calls whose workspace and outputs land on memory an earlier call used
for something else (the caching allocator recycles blocks).  The postscan is a
programmatic dependent launch: its reads of the prescan's records and range
histograms must not be served from lines an earlier kernel left in L1
(regression: the m > 32 pipeline returned wrong offsets on the second call
while every single-call parity test passed)."""
import numpy as np
import pytest
import torch

import oracle
from gen import device as gdev
from gen import inputs as gen

pytestmark = pytest.mark.gpu
ms = pytest.importorskip("paper_1701_01189_b200")


def host(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("pairs", [False, True])
def test_repeated_calls_recycled_memory(pairs):
    n = 1 << 24
    ms.device_init(0)
    cases = []
    for m in (256, 64, 128, 256, 32, 256, 8, 256):
        k = torch.empty(n, dtype=torch.int32, device="cuda")
        gdev.keys_(k, 11 + m, kind=gen.IDENTITY, m=m)
        cases.append((m, k))
    v = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.values_(v, 5, parity=True)
    vh = host(v)
    for m, k in cases:
        ek, ev, eo = oracle.multisplit(host(k), oracle.identity(m), vh if pairs else None)
        for _ in range(3):
            ko, vo, off = ms.multisplit(k, v if pairs else None, bucket=ms.Identity(m))
            assert np.array_equal(host(off), eo), f"m={m}"
            assert np.array_equal(host(ko), ek), f"m={m}"
            if pairs:
                assert np.array_equal(host(vo), ev), f"m={m}"
            del ko, vo, off
            torch.cuda.empty_cache() if m == 64 else None


def test_sort_repeated_8bit():
    """The 4 x 8-bit sort: four m = 256 calls back to back on one workspace, twice."""
    n = 1 << 22
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(k, 3)
    ek, _ = oracle.radix_sort(host(k))
    for _ in range(3):
        ko, _ = ms.radix_sort(k, bits_per_pass=8)
        assert np.array_equal(host(ko), ek)
