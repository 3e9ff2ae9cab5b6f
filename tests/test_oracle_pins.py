"""Pins for the CPU oracle (oracle/): each check ties the oracle to something
other than itself -- the paper's definitions written as brute force, worked
examples (tests/golden, cited), exhaustive small alphabets, library routines
for special cases, and invariants -- so that a dropped term, a wrong sign or
index, or a transposed operand in the oracle fails at least one of them.
"""
import itertools

import numpy as np
import pytest

import oracle
from gen import inputs as gen
from tests.conftest import golden, golden_kv, ints, matrix


def eq1_positions(b: np.ndarray) -> np.ndarray:
    """Eq.(1) evaluated literally, O(n^2):
    p(i) = |{r : f(u_r) < f(u_i)}| + |{r < i : f(u_r) = f(u_i)}|."""
    n = b.size
    p = np.empty(n, np.int64)
    for i in range(n):
        p[i] = int(np.count_nonzero(b < b[i])) + int(np.count_nonzero(b[:i] == b[i]))
    return p


def buckets(keys, fn):
    return np.array([oracle.bucket_of(fn, int(k)) for k in keys], np.int64)


# --------------------------------------------------------------------------- bucket functions

def test_bucket_spec_examples():
    # Delta(100), key 250 -> 2 ; RadixBits(k=1, r=4), 0xAB -> 0xA
    assert oracle.bucket_of(oracle.delta(256, 100), 250) == 2
    assert oracle.bucket_of(oracle.radix(4, 4), 0xAB) == 0xA


@pytest.mark.parametrize("d", [1, 2, 3, 7, 100, 2**31 - 1, 2**31, 2**31 + 1, 2**32 - 1])
def test_delta_bucket_edges(d):
    # Delta buckets partition the key domain into [bD, (b+1)D); keys beyond
    # (m-1)D clamp into m-1 (reading R7).  Checked at every bucket edge.
    m = 256
    fn = oracle.delta(m, d)
    for b in range(1, m):
        lo = b * d
        if lo > 0xFFFFFFFF:
            break
        assert oracle.bucket_of(fn, lo) == b
        assert oracle.bucket_of(fn, lo - 1) == b - 1
    assert oracle.bucket_of(fn, 0) == 0
    assert oracle.bucket_of(fn, 0xFFFFFFFF) == min(0xFFFFFFFF // d, m - 1)


@pytest.mark.parametrize("m", list(range(1, 257)))
def test_delta_default_width(m):
    # default D = ceil(2^32/m): every key lands in [0, m), bucket edges at multiples of D,
    # and for power-of-two m the bucket is the top log2(m) bits (closed form).
    fn = oracle.delta(m)
    d = fn.delta
    assert oracle.bucket_of(fn, 0xFFFFFFFF) == m - 1
    if m > 1:
        assert oracle.bucket_of(fn, d - 1) == 0 and oracle.bucket_of(fn, d) == 1
        assert oracle.bucket_of(fn, (m - 1) * d) == m - 1
        assert oracle.bucket_of(fn, (m - 1) * d - 1) == m - 2
    if m & (m - 1) == 0 and m > 1:
        k = m.bit_length() - 1
        for u in (0, 1, 12345, 0x80000000, 0xDEADBEEF, 0xFFFFFFFF):
            assert oracle.bucket_of(fn, u) == u >> (32 - k)


def test_radix_bucket_bits():
    rng = np.random.default_rng(5)
    for u in rng.integers(0, 2**32, 50, dtype=np.uint64):
        u = int(u)
        digits = [oracle.bucket_of(oracle.radix(8 * k, 8), u) for k in range(4)]
        assert sum(dk << (8 * k) for k, dk in enumerate(digits)) == u  # the 4 digits rebuild u
        assert oracle.bucket_of(oracle.radix(0, 1), u) == u % 2


def test_identity_domain_and_validation():
    assert oracle.bucket_of(oracle.identity(8), 7) == 7
    with pytest.raises(oracle.OracleError) as e:
        oracle.bucket_of(oracle.identity(8), 8)
    assert e.value.code == oracle.ERR_KEY_DOMAIN
    with pytest.raises(oracle.OracleError):
        oracle.multisplit([0, 1, 9], oracle.identity(8))
    assert oracle.validate(oracle.Bucket(oracle.DELTA, 4, delta=0)) == oracle.ERR_INVALID
    assert oracle.validate(oracle.Bucket(oracle.IDENTITY, 0)) == oracle.ERR_UNSUPPORTED
    # m > 256 is the extended regime of Sec.6.3, up to 65536 buckets
    assert oracle.validate(oracle.Bucket(oracle.IDENTITY, 257)) == oracle.OK
    assert oracle.validate(oracle.Bucket(oracle.IDENTITY, 65537)) == oracle.ERR_UNSUPPORTED
    assert oracle.validate(oracle.Bucket(oracle.RADIX, 256, shift=25, bits=8)) == oracle.ERR_INVALID
    assert oracle.validate(oracle.Bucket(oracle.RADIX, 128, shift=0, bits=8)) == oracle.ERR_INVALID
    assert oracle.validate(oracle.radix(24, 8)) == oracle.OK


# --------------------------------------------------------------------------- multisplit (Eq.1)

def test_worked_example_s219():
    g = golden_kv("spec_s219_identity_m4.txt")
    keys = ints(g["keys"])
    ko, _, off = oracle.multisplit(keys, oracle.identity(int(g["m"])))
    assert ko.tolist() == ints(g["keys_out"])
    assert off.tolist() == ints(g["offsets"])
    p = ints(g["p"])
    assert eq1_positions(np.array(keys)).tolist() == p
    assert [ko[pi] for pi in p] == keys


def test_fig_localization_matrix_local_offsets():
    # B_j at positions {1,4,5,8,11,14} of a 16-element subproblem -> local
    # offsets 0..5 and count 6.  Build it with delta m=2 (B_j = bucket 1).
    g = golden_kv("paper_fig_localization_matrix.txt")
    n, pos = int(g["n"]), ints(g["positions"])
    fn = oracle.delta(2)
    keys = np.full(n, 5, np.uint32)
    keys[pos] = 0x80000000 + np.arange(len(pos), dtype=np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, off = oracle.multisplit(keys, fn, vals)
    start, end = int(off[1]), int(off[2])
    assert end - start == int(g["count"])
    # local offset of input element i = (its output position) - (bucket start)
    where = {int(v): k for k, v in enumerate(vo)}
    assert [where[i] - start for i in pos] == ints(g["local_offsets"])


def test_spec_window_examples_as_local_offsets():
    # SPEC S:165-166 (Alg.3 results): all-same bucket -> offset i; alternating 0,1 -> floor(i/2)
    lane = np.arange(32, dtype=np.uint32)
    for ids, expect in ((np.zeros(32, np.uint32), lane), (lane % 2, lane // 2)):
        _, vo, off = oracle.multisplit(ids, oracle.identity(2), lane)
        local = np.empty(32, np.int64)
        for pos, i in enumerate(vo):
            local[i] = pos - off[ids[i]]
        assert local.tolist() == expect.tolist()


@pytest.mark.parametrize("m", [1, 2, 3])
def test_exhaustive_small_alphabets(m):
    # every key sequence over [0,m) with n <= 7 (3^7 = 2187 sequences at m=3):
    # oracle == Eq.(1) brute force == Python's stable sorted() (identity key-only = sort)
    fn = oracle.identity(m)
    for n in range(0, 8):
        for seq in itertools.product(range(m), repeat=n):
            keys = np.array(seq, np.uint32)
            vals = np.arange(n, dtype=np.uint32)
            ko, vo, off = oracle.multisplit(keys, fn, vals)
            p = eq1_positions(keys.astype(np.int64))
            exp_k = np.empty(n, np.uint32)
            exp_v = np.empty(n, np.uint32)
            exp_k[p] = keys
            exp_v[p] = vals
            assert ko.tolist() == exp_k.tolist() == sorted(seq)
            assert vo.tolist() == exp_v.tolist() == sorted(range(n), key=lambda i: seq[i])
            assert off.tolist() == [sum(1 for s in seq if s < j) for j in range(m + 1)]


@pytest.mark.parametrize("case", [(oracle.delta(2), 300), (oracle.delta(7), 700),
                                  (oracle.delta(256), 1500), (oracle.radix(4, 5), 2048),
                                  (oracle.identity(33), 1000)])
def test_eq1_brute_force_random(case):
    fn, n = case
    kind = fn.kind
    keys = gen.keys(n, seed=11, kind=kind, m=fn.m, delta=fn.delta, shift=fn.shift, bits=fn.bits,
                    dist=gen.DIST_SKEW, alpha=0.5)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, _ = oracle.multisplit(keys, fn, vals)
    p = eq1_positions(buckets(keys, fn))
    assert np.array_equal(ko[p], keys)
    assert np.array_equal(vo[p], vals)


@pytest.mark.parametrize("k", [1, 3, 5, 8])
def test_special_cases_library_routines(k):
    rng = np.random.default_rng(k)
    keys = rng.integers(0, 2**32, 5000, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(keys.size, dtype=np.uint32)
    # DELTA with m = 2^k and D = 2^(32-k)  ==  stable sort by u >> (32-k)
    ko, vo, _ = oracle.multisplit(keys, oracle.delta(1 << k), vals)
    order = np.argsort(keys >> np.uint32(32 - k), kind="stable")
    assert np.array_equal(ko, keys[order]) and np.array_equal(vo, order.astype(np.uint32))
    # RADIX(s, r)  ==  stable sort by (u >> s) & (2^r - 1)
    s = 32 - k - 2
    ko, vo, _ = oracle.multisplit(keys, oracle.radix(s, k), vals)
    order = np.argsort((keys >> np.uint32(s)) & np.uint32((1 << k) - 1), kind="stable")
    assert np.array_equal(ko, keys[order]) and np.array_equal(vo, order.astype(np.uint32))
    # IDENTITY key-only  ==  sort
    small = (keys % np.uint32(1 << k)).astype(np.uint32)
    ko, _, _ = oracle.multisplit(small, oracle.identity(1 << k))
    assert np.array_equal(ko, np.sort(small))


def test_m1_and_single_bucket_are_copies():
    keys = gen.keys(999, seed=3)
    vals = gen.values(999, seed=3)
    ko, vo, off = oracle.multisplit(keys, oracle.delta(1), vals)
    assert np.array_equal(ko, keys) and np.array_equal(vo, vals) and off.tolist() == [0, 999]
    fn = oracle.delta(64)
    one = gen.keys(999, seed=3, kind=gen.DELTA, m=64, delta=fn.delta, dist=gen.DIST_SKEW, alpha=0.0)
    ko, vo, _ = oracle.multisplit(one, fn, vals)
    assert np.array_equal(ko, one) and np.array_equal(vo, vals)


def test_empty_input():
    # keys=[], m=5 -> empty output, offsets all zero
    ko, vo, off = oracle.multisplit(np.zeros(0, np.uint32), oracle.identity(5), np.zeros(0, np.uint32))
    assert ko.size == 0 and vo.size == 0 and off.tolist() == [0] * 6


@pytest.mark.parametrize("dist", [gen.DIST_UNIFORM, gen.DIST_SKEW, gen.DIST_BINOMIAL])
@pytest.mark.parametrize("m", [2, 33, 256])
def test_invariants(dist, m):
    # permutation, non-decreasing bucket ids, stability, offsets = counts
    n = 20000
    fn = oracle.delta(m)
    keys = gen.keys(n, seed=m, kind=gen.DELTA, m=m, delta=fn.delta, dist=dist)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, off = oracle.multisplit(keys, fn, vals)
    b_in = (keys.astype(np.uint64) // np.uint64(fn.delta)).clip(0, m - 1)
    b_out = (ko.astype(np.uint64) // np.uint64(fn.delta)).clip(0, m - 1)
    assert np.array_equal(np.sort(ko), np.sort(keys))
    assert np.array_equal(keys[vo], ko)
    assert np.all(np.diff(b_out.astype(np.int64)) >= 0)
    same = b_out[1:] == b_out[:-1]
    assert np.all(vo[1:][same] > vo[:-1][same])
    assert np.array_equal(np.diff(off.astype(np.int64)), np.bincount(b_in.astype(np.int64), minlength=m))
    assert off[0] == 0 and off[m] == n


# --------------------------------------------------------------------------- H and G (Eq.2)

def test_prescan_example_s183():
    g = golden_kv("spec_s183_prescan.txt")
    H = oracle.tile_histogram(ints(g["keys"]), oracle.identity(int(g["m"])), T=4)
    assert H.T.tolist() == matrix(g["H"])


def test_warp_histogram_examples():
    # SPEC S:156-158 as one 32-element subproblem (T = 32)
    lane = np.arange(32, dtype=np.uint32)
    assert oracle.tile_histogram(np.zeros(32, np.uint32), oracle.identity(2), 32)[0].tolist() == [32, 0]
    assert oracle.tile_histogram(lane % 4, oracle.identity(4), 32)[0].tolist() == [8, 8, 8, 8]
    h = oracle.tile_histogram(lane * 2, oracle.identity(64), 32)[0]
    assert h[0::2].tolist() == [1] * 32 and h[1::2].tolist() == [0] * 32


def test_prescan_column_sums_s184():
    # n=448 keys, subproblems of 224 -> 2 columns, column sums [224, 224]
    keys = gen.keys(448, seed=1)
    H = oracle.tile_histogram(keys, oracle.delta(8), 224)
    assert H.shape == (2, 8) and H.sum(axis=1).tolist() == [224, 224]


@pytest.mark.parametrize("T", [1, 7, 32, 1000, 4096, 10**6])
def test_tile_histogram_vs_bincount(T):
    n, m = 9001, 37
    fn = oracle.delta(m)
    keys = gen.keys(n, seed=T, kind=gen.DELTA, m=m, delta=fn.delta, dist=gen.DIST_BINOMIAL)
    b = (keys.astype(np.uint64) // np.uint64(fn.delta)).clip(0, m - 1).astype(np.int64)
    H = oracle.tile_histogram(keys, fn, T)
    L = -(-n // T)
    assert H.shape == (L, m)
    for l in range(L):
        assert H[l].tolist() == np.bincount(b[l * T:(l + 1) * T], minlength=m).tolist()


def test_global_scan_examples_s192():
    rows = golden("spec_s192_scan.txt")
    for hline, gline in zip(rows[0::2], rows[1::2]):
        Hm = np.array(matrix(hline.split(":", 1)[1]), np.uint32)  # m x L
        Gm = np.array(matrix(gline.split(":", 1)[1]), np.uint32)
        assert oracle.global_scan(Hm.T.copy()).T.tolist() == Gm.tolist()


def test_global_scan_vs_cumsum():
    rng = np.random.default_rng(2)
    H = rng.integers(0, 1000, (123, 45), dtype=np.uint64).astype(np.uint32)  # [L, m]
    row = H.T.reshape(-1).astype(np.int64)                                    # bucket-major
    excl = np.concatenate([[0], np.cumsum(row)[:-1]])
    assert np.array_equal(oracle.global_scan(H).T.reshape(-1).astype(np.int64), excl)


@pytest.mark.parametrize("T", [1, 5, 64, 333])
def test_eq2_equals_eq1(T):
    # Eq.(2): p(i) = G[b][l] + |{r in subproblem l, r < i, same bucket}|
    # must reproduce the oracle's Eq.(1) permutation for every element.
    n, m = 2000, 9
    fn = oracle.delta(m)
    keys = gen.keys(n, seed=T, kind=gen.DELTA, m=m, delta=fn.delta, dist=gen.DIST_SKEW, alpha=0.3)
    b = buckets(keys, fn)
    G = oracle.global_scan(oracle.tile_histogram(keys, fn, T))
    vals = np.arange(n, dtype=np.uint32)
    _, vo, _ = oracle.multisplit(keys, fn, vals)
    pos = np.empty(n, np.int64)
    pos[vo] = np.arange(n)
    for i in range(n):
        l = i // T
        local = int(np.count_nonzero(b[l * T:i] == b[i]))
        assert int(G[l, b[i]]) + local == pos[i]


# --------------------------------------------------------------------------- radix sort (Sec.7.1)

@pytest.mark.parametrize("bounds", [(0, 32), (0, 8), (4, 20), (24, 32), (31, 32)])
def test_radix_sort_vs_numpy_stable(bounds):
    lo, hi = bounds
    rng = np.random.default_rng(hi)
    keys = rng.integers(0, 2**32, 30000, dtype=np.uint64).astype(np.uint32)
    keys[::3] = keys[::3] & np.uint32(0x00FF00FF)  # many duplicates -> stability visible
    vals = np.arange(keys.size, dtype=np.uint32)
    mask = np.uint64((1 << (hi - lo)) - 1)
    order = np.argsort((keys.astype(np.uint64) >> np.uint64(lo)) & mask, kind="stable")
    ko, vo = oracle.radix_sort(keys, vals, lo, hi)
    assert np.array_equal(ko, keys[order]) and np.array_equal(vo, order.astype(np.uint32))


@pytest.mark.parametrize("r", [4, 7, 8])
def test_radix_sort_equals_lsd_multisplit_passes(r):
    # ceil(32/r) LSD passes of stable multisplit with f_k(u)=(u>>kr)&(2^r-1)
    # (last pass narrower) produce the sorted output.
    rng = np.random.default_rng(r)
    keys = rng.integers(0, 2**32, 4000, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(keys.size, dtype=np.uint32)
    k, v = keys, vals
    for shift in range(0, 32, r):
        k, v, _ = oracle.multisplit(k, oracle.radix(shift, min(r, 32 - shift)), v)
    ko, vo = oracle.radix_sort(keys, vals)
    assert np.array_equal(k, ko) and np.array_equal(v, vo)
    assert np.all(np.diff(ko.astype(np.int64)) >= 0)


# --------------------------------------------------------------------------- generators

def test_splitmix64_reference_values():
    # splitmix64 of state 0: first two outputs of the published generator
    z = gen.mix64(np.array([0, 0x9E3779B97F4A7C15], np.uint64))
    assert [int(x) for x in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]


def test_generator_chunk_independence():
    a = gen.keys(gen._CHUNK + 17, seed=9, kind=gen.RADIX, m=256, shift=8, bits=8, dist=gen.DIST_SKEW)
    b = gen.keys(40, seed=9, kind=gen.RADIX, m=256, shift=8, bits=8, dist=gen.DIST_SKEW)
    assert np.array_equal(a[:40], b)


def test_generator_skew_share():
    # alpha-uniform: hot bucket share 0.9 + 0.1/m for alpha = 0.1 (within 5 sigma)
    n, m = 200000, 128
    fn = oracle.delta(m)
    keys = gen.keys(n, seed=4, kind=gen.DELTA, m=m, delta=fn.delta, dist=gen.DIST_SKEW, alpha=0.1)
    counts = np.bincount((keys.astype(np.uint64) // np.uint64(fn.delta)).astype(np.int64), minlength=m)
    p = 0.9 + 0.1 / m
    assert abs(counts.max() / n - p) < 5 * np.sqrt(p * (1 - p) / n)


def test_generator_binomial_empty_buckets():
    # B(m-1, 1/2): expected empty buckets = sum_k (1 - C(m-1,k)/2^(m-1))^n exactly
    # (reading R16: the paper's "almost 184" at n=2^25 does not match this expectation).
    from math import comb
    n, m = 1 << 18, 256
    expect = sum((1 - comb(m - 1, k) / 2 ** (m - 1)) ** n for k in range(m))
    b = gen.keys(n, seed=6, kind=gen.IDENTITY, m=m, dist=gen.DIST_BINOMIAL)
    empty = m - np.count_nonzero(np.bincount(b.astype(np.int64), minlength=m))
    assert abs(empty - expect) <= 3
    assert abs(b.mean() - (m - 1) / 2) < 0.05
    e25 = sum((1 - comb(m - 1, k) / 2 ** (m - 1)) ** (1 << 25) for k in range(m))
    assert 169 < e25 < 170.5


def test_metric_definitions_sol():
    # SOL = BW / 12 B (keys) and BW / 20 B (pairs); Table timing vs ms_rate
    rows = [ln for ln in golden("paper_sol.txt") if not ln.startswith("n=")]
    for ln in rows:
        bw, ks, ps = (float(x) for x in ln.split())
        assert abs(bw / 12 - ks) < 0.1 and abs(bw / 20 - ps) < 0.1
    n = 2**25
    assert abs(n / 1.77e-3 / 1e9 - 18.93) < 0.05


# ---------------------------------------------------------------- histogram (Sec.7.3)
def _hist_edge_samples(s):
    """samples on and next to every splitter, outside the range, NaN, and the grid."""
    s = np.asarray(s, np.float32)
    pts = [s, np.nextafter(s, np.float32(-np.inf)), np.nextafter(s, np.float32(np.inf)),
           np.array([-1.0, -0.0, 2048.0, np.nan, np.inf, -np.inf], np.float32)]
    return np.concatenate(pts + [gen.floats(5000, seed=4)]).astype(np.float32)


@pytest.mark.parametrize("m", [1, 2, 3, 7, 64, 255, 256])
def test_histogram_range_is_searchsorted(m):
    # Range scenario = upper-bound search = numpy.searchsorted(side="right") - 1
    s = gen.splitters(m, seed=m)
    x = _hist_edge_samples(s)
    inside = (x >= s[0]) & (x < s[m])
    b = np.searchsorted(s, x[inside], side="right") - 1
    expect = np.bincount(b, minlength=m).astype(np.uint32)
    assert np.array_equal(oracle.histogram_range(x, s), expect)


@pytest.mark.parametrize("k", [0, 1, 3, 5, 8])
def test_histogram_even_power_of_two_exact(k):
    # Delta = 1024 / 2^k is a power of two: floor((x - 0) / Delta) is exact, so the
    # bucket is integer arithmetic on the sample's grid value x * 2^14 (gen.floats)
    m = 1 << k
    x = gen.floats(20000, seed=9)
    xi = (x.astype(np.float64) * (1 << 14)).astype(np.int64)  # exact integers
    width = (1024 // m) * (1 << 14)
    expect = np.bincount(xi // width, minlength=m).astype(np.uint32)
    assert np.array_equal(oracle.histogram_even(x, m, 0.0, 1024.0), expect)


@pytest.mark.parametrize("k", [1, 4, 8])
def test_histogram_even_equals_range_on_even_splitters(k):
    m = 1 << k
    s = (np.arange(m + 1) * (1024.0 / m)).astype(np.float32)  # exact
    x = _hist_edge_samples(s)
    assert np.array_equal(oracle.histogram_even(x, m, 0.0, 1024.0), oracle.histogram_range(x, s))


@pytest.mark.parametrize("m", [3, 7, 100, 255])
def test_histogram_even_general_m_matches_exact_quotient_off_boundary(m):
    # reading R25: binary32 quotient; away from bucket boundaries it must equal the
    # floor of the exact rational quotient (x - s0) / fl((s_m - s0) / m)
    from fractions import Fraction
    lo, hi = np.float32(0.0), np.float32(1000.0)
    delta = Fraction(float(np.float32((hi - lo) / np.float32(m))))
    x = gen.floats(3000, seed=m) * np.float32(1000.0 / 1024.0)
    c = oracle.histogram_even(x, m, float(lo), float(hi))
    expect = np.zeros(m, np.int64)
    unsure = 0
    for v in x.astype(np.float64):
        q = (Fraction(v) - Fraction(float(lo))) / delta
        fl = q.numerator // q.denominator
        if abs(q - round(q)) < Fraction(1, 10000):
            unsure += 1
            continue
        expect[min(fl, m - 1)] += 1
    assert unsure < 30
    assert int(c.sum()) == x.size
    assert np.all(np.abs(c.astype(np.int64) - expect) <= unsure)


def test_histogram_worked_example():
    # P:1890 with s_0 = 0, s_m = 1024, m = 256 (Delta = 4): 0, 0.5, 3.9 -> bucket 0;
    # 4 -> 1; 1023.99 -> 255; 1024 (= s_m), -1 and NaN are outside [s_0, s_m) (reading R26)
    x = np.array([0, 0.5, 3.9, 4, 1023.99, 1024, -1, np.nan], np.float32)
    c = oracle.histogram_even(x, 256, 0.0, 1024.0)
    assert c[0] == 3 and c[1] == 1 and c[255] == 1 and c.sum() == 5
    r = oracle.histogram_range(x, np.array([0, 1, 4, 1024], np.float32))
    assert r.tolist() == [2, 1, 2]
