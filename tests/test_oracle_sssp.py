"""Pins for the SSSP oracle (Sec.7.2: Dijkstra) and the R-MAT
generator: a hand-checked example, scipy's Dijkstra (a library routine) on
R-MAT graphs, Bellman-Ford-Moore by brute force on graphs with zero
weights, self loops, parallel edges and unreachable vertices, and the
shortest-path optimality conditions."""
import numpy as np
import pytest

import oracle
from gen.graphs import rmat_csr, rmat_edges, to_csr

INF = 0xFFFFFFFF


def csr(V, edges):
    s = np.array([e[0] for e in edges], np.uint32)
    d = np.array([e[1] for e in edges], np.uint32)
    w = np.array([e[2] for e in edges], np.uint32)
    return to_csr(V, s, d, w)


def bellman_ford(V, src, dst, w, source):
    """Bellman-Ford-Moore: relax every edge, V-1 rounds (numpy, brute force)."""
    d = np.full(V, np.iinfo(np.int64).max // 4, np.int64)
    d[source] = 0
    for _ in range(V - 1):
        nd = d[src] + w.astype(np.int64)
        new = d.copy()
        np.minimum.at(new, dst, nd)
        if np.array_equal(new, d):
            break
        d = new
    out = np.where(d >= np.iinfo(np.int64).max // 8, INF, d)
    return out.astype(np.uint32)


def test_hand_example():
    # s=0, t=1, x=2, y=3, z=4 (the classic 5-vertex Dijkstra example); by hand:
    # y = 5 (s->y), z = 7 (s->y->z), t = 8 (s->y->t), x = 9 (s->y->t->x)
    g = csr(5, [(0, 1, 10), (0, 3, 5), (1, 2, 1), (1, 3, 2), (3, 1, 3), (3, 2, 9), (3, 4, 2),
                (2, 4, 4), (4, 2, 6), (4, 0, 7)])
    assert oracle.sssp(*g, 0).tolist() == [0, 8, 9, 5, 7]
    assert oracle.sssp(*g, 2).tolist() == [11, 19, 0, 16, 4]


@pytest.mark.parametrize("scale,ef", [(8, 8), (10, 16), (12, 4)])
def test_rmat_vs_scipy_dijkstra(scale, ef):
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra
    V, s, d, w = rmat_edges(scale, ef, seed=scale)
    w = w + 1  # scipy: strictly positive weights (explicit zeros are ambiguous there)
    keep = s != d
    s, d, w = s[keep], d[keep], w[keep]
    # parallel edges: scipy would sum duplicates, so keep the lightest of each pair
    key = s.astype(np.uint64) << np.uint64(32) | d.astype(np.uint64)
    order = np.lexsort((w, key))
    first = np.ones(order.size, bool)
    first[1:] = key[order][1:] != key[order][:-1]
    s, d, w = s[order][first], d[order][first], w[order][first]
    m = csr_matrix((w.astype(np.float64), (s, d)), shape=(V, V))
    for src in (0, 1, V // 2):
        exp = dijkstra(m, directed=True, indices=src)
        exp = np.where(np.isinf(exp), INF, exp).astype(np.uint64).astype(np.uint32)
        assert np.array_equal(oracle.sssp(*to_csr(V, s, d, w), src), exp)


@pytest.mark.parametrize("seed", range(6))
def test_bellman_ford_brute_force(seed):
    r = np.random.default_rng(seed)
    V = int(r.integers(1, 60))
    E = int(r.integers(0, 4 * V))
    s = r.integers(0, V, E).astype(np.uint32)
    d = r.integers(0, V, E).astype(np.uint32)
    w = r.integers(0, 4, E).astype(np.uint32)  # many zero weights, ties, parallel edges, loops
    src = int(r.integers(0, V))
    assert np.array_equal(oracle.sssp(*to_csr(V, s, d, w), src), bellman_ford(V, s, d, w, src))


def test_optimality_conditions_rmat():
    V, rp, col, w = rmat_csr(11, 8, seed=3)
    dist = oracle.sssp(rp, col, w, 0).astype(np.int64)
    src = np.repeat(np.arange(V), np.diff(rp.astype(np.int64)))
    reach = dist[src] != INF
    # no edge can still be relaxed, and every reached vertex but the source has a tight edge
    assert np.all(dist[col[reach]] <= dist[src[reach]] + w[reach])
    tight = np.zeros(V, bool)
    ok = reach & (dist[col] == dist[src] + w)
    tight[col[ok]] = True
    reached = dist != INF
    reached[0] = False
    assert np.all(tight[reached]) and dist[0] == 0


def test_rmat_generator_shape():
    V, s, d, w = rmat_edges(10, 16, seed=1)
    assert V == 1024 and s.size == 16384 and w.max() <= 1000
    # vertex 0 is the source of an edge iff every level picks row 0 (probability a + b = 0.6):
    # its out-degree is binomial(E, 0.6^scale), mean 99.0 here, checked within 5 sigma
    deg = np.bincount(s, minlength=V)
    mu = 16384 * 0.6 ** 10
    assert abs(deg[0] - mu) < 5 * np.sqrt(mu) and deg.max() == deg[0]
    # the column bit is 1 with probability b + d = 0.4 per level (row bit c + d = 0.4)
    assert abs(((d >> 9) & 1).mean() - 0.4) < 0.03 and abs(((s >> 9) & 1).mean() - 0.4) < 0.03


def test_invalid_and_unrepresentable():
    g = csr(2, [(0, 1, 5)])
    with pytest.raises(oracle.OracleError):
        oracle.sssp(*g, 2)
    big = csr(3, [(0, 1, 0xFFFFFFF0), (1, 2, 0x20)])
    with pytest.raises(oracle.OracleError):
        oracle.sssp(*big, 0)
    assert oracle.sssp(*csr(3, [(1, 2, 1)]), 0).tolist() == [0, INF, INF]
