"""GPU parity of the device-wide histogram (Sec.7.3) against the
oracle: bit-exact counts for Even and Range scenarios, m = 1..256, on the
paper's samples (U[0,1024) binary32) plus edge samples (every splitter
and its neighbouring floats, out-of-range values, NaN, infinities), ragged
sizes, unaligned sample pointers and the full size n = 2^25."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gen

pytestmark = pytest.mark.gpu

ms = pytest.importorskip("paper_1701_01189_b200")


def edges(s):
    s = np.asarray(s, np.float32)
    return np.concatenate([s, np.nextafter(s, np.float32(-np.inf)), np.nextafter(s, np.float32(np.inf)),
                           np.array([-1.0, -0.0, 2048.0, np.nan, np.inf, -np.inf], np.float32)])


def host(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("m", [1, 2, 3, 8, 32, 33, 100, 255, 256])
@pytest.mark.parametrize("n", [0, 1, 1000, 4097, (1 << 20) + 3])
def test_even(m, n):
    x = gen.floats(n, seed=m + n)
    s = (np.arange(m + 1) * (1024.0 / m)).astype(np.float32)
    x = np.concatenate([x, edges(s)]) if n else x
    got = host(ms.histogram_even(torch.from_numpy(x).cuda(), m, 0.0, 1024.0))
    assert np.array_equal(got, oracle.histogram_even(x, m, 0.0, 1024.0))


@pytest.mark.parametrize("m", [1, 2, 3, 8, 32, 33, 100, 255, 256])
@pytest.mark.parametrize("n", [0, 1, 1000, 4097, (1 << 20) + 3])
def test_range(m, n):
    s = gen.splitters(m, seed=m)
    x = gen.floats(n, seed=2 * m + n)
    x = np.concatenate([x, edges(s)]) if n else x
    got = host(ms.histogram_range(torch.from_numpy(x).cuda(), torch.from_numpy(s).cuda()))
    assert np.array_equal(got, oracle.histogram_range(x, s))


@pytest.mark.parametrize("lo,hi,m", [(0.0, 1000.0, 7), (-3.5, 17.25, 100), (1e-3, 1e3, 255)])
def test_even_general_bounds(lo, hi, m):
    x = (gen.floats(300000, seed=5) * np.float32((hi - lo) / 1024.0) + np.float32(lo)).astype(np.float32)
    got = host(ms.histogram_even(torch.from_numpy(x).cuda(), m, lo, hi))
    assert np.array_equal(got, oracle.histogram_even(x, m, lo, hi))


def test_unaligned_samples():
    x = gen.floats(100003, seed=3)
    xd = torch.from_numpy(x).cuda()
    for off in (1, 2, 3):
        got = host(ms.histogram_even(xd[off:], 64, 0.0, 1024.0))
        assert np.array_equal(got, oracle.histogram_even(x[off:], 64, 0.0, 1024.0))


def test_full_size_and_errors():
    n = 1 << 25
    x = gen.floats(n, seed=0x5EED)
    xd = torch.from_numpy(x).cuda()
    for m in (2, 256):
        assert np.array_equal(host(ms.histogram_even(xd, m, 0.0, 1024.0)), oracle.histogram_even(x, m, 0.0, 1024.0))
    s = gen.splitters(256, seed=1)
    assert np.array_equal(host(ms.histogram_range(xd, torch.from_numpy(s).cuda())), oracle.histogram_range(x, s))
    with pytest.raises(Exception):
        ms.histogram_even(xd, 257, 0.0, 1024.0)
    with pytest.raises(Exception):
        ms.histogram_even(xd, 8, 1.0, 1.0)
