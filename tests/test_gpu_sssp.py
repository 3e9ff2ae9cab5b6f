"""GPU parity of Multisplit-SSSP (Sec.7.2) against the oracle's
Dijkstra: distances bit-exact on R-MAT graphs and on graphs with zero
weights, self loops, parallel edges, unreachable parts, one vertex, no edges."""
import numpy as np
import pytest
import torch

import oracle
from gen.graphs import rmat_csr, to_csr

pytestmark = pytest.mark.gpu
ms = pytest.importorskip("paper_1701_01189_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def run(rp, col, w, src, **kw):
    return ms.sssp(dev(rp), dev(col), dev(w), src, **kw).cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("scale,ef", [(6, 4), (10, 16), (14, 8), (16, 16)])
@pytest.mark.parametrize("delta,K", [(100, 10), (1, 10), (1000, 2), (37, 256), (1 << 30, 10), (50, 1)])
def test_rmat(scale, ef, delta, K):
    V, rp, col, w = rmat_csr(scale, ef, seed=scale * 31 + ef)
    for src in (0, V - 1):
        exp = oracle.sssp(rp, col, w, src)
        got = run(rp, col, w, src, delta=delta, buckets=K)
        assert np.array_equal(got, exp), f"src={src}"


@pytest.mark.parametrize("seed", range(8))
def test_random_small_graphs(seed):
    r = np.random.default_rng(seed)
    V = int(r.integers(1, 3000))
    E = int(r.integers(0, 8 * V))
    s = r.integers(0, V, E).astype(np.uint32)
    d = r.integers(0, V, E).astype(np.uint32)
    w = r.integers(0, [1, 3, 1000, 100000][seed % 4] + 1, E).astype(np.uint32)  # zero weights included
    rp, col, w = to_csr(V, s, d, w)
    src = int(r.integers(0, V))
    assert np.array_equal(run(rp, col, w, src, delta=int(r.integers(1, 500))), oracle.sssp(rp, col, w, src))


def test_degenerate():
    rp, col, w = to_csr(1, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    assert run(rp, col, w, 0).tolist() == [0]
    rp, col, w = to_csr(4, np.array([1, 2], np.uint32), np.array([2, 3], np.uint32), np.array([5, 5], np.uint32))
    assert run(rp, col, w, 0).tolist() == [0, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF]
    assert run(rp, col, w, 1).tolist() == [0xFFFFFFFF, 0, 5, 10]
    # a hub of degree >= 32 (warp-wide expansion) next to degree-1 vertices, parallel edges
    s = np.array([0] * 100 + list(range(1, 100)) + [5, 5], np.uint32)
    d = np.array(list(range(1, 101)) + list(range(2, 101)) + [7, 7], np.uint32)
    w = np.arange(s.size, dtype=np.uint32) % 13
    rp, col, w = to_csr(101, s, d, w)
    assert np.array_equal(run(rp, col, w, 0, delta=3), oracle.sssp(rp, col, w, 0))


def test_stats_and_errors():
    V, rp, col, w = rmat_csr(12, 8, seed=1)
    d, st = ms.sssp(dev(rp), dev(col), dev(w), 0, stats=True)
    assert st["iterations"] >= 1 and st["frontier"] <= st["items"]
    with pytest.raises(ms.MultisplitError):
        ms.sssp(dev(rp), dev(col), dev(w), V)  # source out of range
    with pytest.raises(ms.MultisplitError):
        ms.sssp(dev(rp), dev(col), dev(w), 0, delta=0)
