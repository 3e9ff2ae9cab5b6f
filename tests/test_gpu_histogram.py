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


@pytest.mark.parametrize("layout", ["crowded", "half_crowded", "huge_span", "tiny_span", "geometric", "cell_edges"])
@pytest.mark.parametrize("m", [8, 256])
def test_range_cell_table(layout, m):
    """Range cells (1024 cells of [s_0, s_m)): crowded cells take the search, a span
    that overflows binary32 disables the table, cell boundaries are exact."""
    r = np.random.default_rng(m + len(layout))
    if layout == "crowded":         # every interior splitter within one cell
        s = np.concatenate([[0.0], np.sort(r.uniform(500.0, 500.5, m - 1)), [1024.0]])
    elif layout == "half_crowded":
        a = np.sort(r.uniform(3.0, 3.01, (m - 1) // 2))
        b = np.sort(r.uniform(10.0, 1000.0, m - 1 - a.size))
        s = np.concatenate([[0.0], a, b, [1024.0]])
    elif layout == "huge_span":     # s_m - s_0 overflows binary32
        s = np.concatenate([[-3.0e38], np.sort(r.uniform(-1e38, 1e38, m - 1)), [3.0e38]])
    elif layout == "tiny_span":     # a few ulps wide
        s = np.float32(1.0) + np.arange(m + 1, dtype=np.float32) * np.float32(2.0 ** -23)
    elif layout == "geometric":     # log-spaced: many splitters in the low cells
        s = np.concatenate([[0.0], np.geomspace(1e-6, 1000.0, m - 1), [1024.0]])
    else:                           # interior splitters exactly on cell starts (s_0 = 0, s_m = 1024)
        s = np.concatenate([[0.0], np.sort(r.choice(np.arange(1, 1024), m - 1, replace=False)).astype(np.float64),
                            [1024.0]])
    s = np.unique(np.asarray(s, np.float32))
    if s.size < 2:
        pytest.skip("degenerate splitters")
    x = np.concatenate([gen.floats(200003, seed=m) * np.float32((s[-1] - s[0]) / 1024.0 if np.isfinite(s[-1] - s[0]) else 1.0)
                        + s[0], edges(s), r.uniform(float(s[0]), float(s[-1]), 5000).astype(np.float32)]).astype(np.float32)
    got = host(ms.histogram_range(torch.from_numpy(x).cuda(), torch.from_numpy(s).cuda()))
    assert np.array_equal(got, oracle.histogram_range(x, s))
