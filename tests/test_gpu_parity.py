"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, on the same seeded inputs.  Integer work => bit-exact.

Grid: SPEC acceptance grid m in {1,2,3,8,32,33,64,255,256} x
n in {0,1,31,32,33,1000,2^20}, plus tile-boundary sizes (ragged tails), the
three bucket identifiers, keys and pairs, uniform / skewed / single-bucket /
binomial inputs; stage-level checks of H and G; radix sort; full-size
configurations of BASELINE.json in the launch configuration bench.py times.
"""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gen

pytestmark = pytest.mark.gpu

ms = pytest.importorskip("paper_1701_01189_b200")


def dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def bucket_pair(kind: str, m: int):
    """(oracle bucket, product bucket, generator kwargs)"""
    if kind == "delta":
        o = oracle.delta(m)
        return o, ms.Delta(m), dict(kind=gen.DELTA, m=m, delta=o.delta)
    if kind == "identity":
        return oracle.identity(m), ms.Identity(m), dict(kind=gen.IDENTITY, m=m)
    bits = max(1, (m - 1).bit_length())
    shift = 32 - bits - 3
    return oracle.radix(shift, bits), ms.Radix(shift, bits), dict(kind=gen.RADIX, m=1 << bits,
                                                                     shift=shift, bits=bits)


def check_multisplit(keys, vals, ob, pb):
    ek, ev, eo = oracle.multisplit(keys, ob, vals)
    ko, vo, off = ms.multisplit(dev(keys), None if vals is None else dev(vals), bucket=pb)
    assert np.array_equal(host(ko), ek), "keys differ"
    if vals is not None:
        assert np.array_equal(host(vo), ev), "values differ"
    assert np.array_equal(host(off), eo), "bucket offsets differ"
    assert ms.device_status() == 0


GRID_M = [1, 2, 3, 8, 32, 33, 64, 255, 256]
GRID_N = [0, 1, 31, 32, 33, 1000, 1 << 20]


@pytest.mark.parametrize("m", GRID_M)
@pytest.mark.parametrize("n", GRID_N)
@pytest.mark.parametrize("pairs", [False, True])
def test_spec_grid_delta(m, n, pairs):
    ob, pb, gk = bucket_pair("delta", m)
    keys = gen.keys(n, seed=1 + m, **gk)
    check_multisplit(keys, gen.values(n, seed=1) if pairs else None, ob, pb)


@pytest.mark.parametrize("kind", ["identity", "radix"])
@pytest.mark.parametrize("m", GRID_M)
@pytest.mark.parametrize("n", [33, 1000, 1 << 20])
def test_spec_grid_identity_radix(kind, m, n):
    if kind == "radix" and m == 1:
        pytest.skip("radix digits have m = 2^bits >= 2")
    ob, pb, gk = bucket_pair(kind, m)
    keys = gen.keys(n, seed=2, dist=gen.DIST_UNIFORM, **gk)
    check_multisplit(keys, gen.values(n, seed=2), ob, pb)


T = 8192  # ms.tile_size() for keys (4096 for pairs); checked below


def test_tile_size():
    assert [ms.tile_size(m, p) for m in (2, 32, 33, 64, 65, 256) for p in (False, True)] == \
        [T, T // 2, T, T // 2, T // 2, T // 2, T // 2, T // 2, T // 2, T // 2, T // 2, T // 2]


@pytest.mark.parametrize("k", [(1, -1), (1, 0), (1, 1), (2, -3), (3, 5), (37, 4097)])
@pytest.mark.parametrize("m", [2, 5, 32, 33, 256])
def test_tile_boundaries_keys(k, m):
    """key-only inputs at exact multiples of the keys tile (ms.tile_size) +- a ragged tail"""
    Tk = ms.tile_size(m, False)
    n = k[0] * Tk + k[1]
    ob, pb, gk = bucket_pair("delta", m)
    keys = gen.keys(n, seed=n + m, dist=gen.DIST_UNIFORM, **gk)
    check_multisplit(keys, None, ob, pb)


@pytest.mark.parametrize("n", [T - 1, T, T + 1, 2 * T - 3, 3 * T + 5, 37 * T + 4097])
@pytest.mark.parametrize("m", [2, 5, 32, 33, 64, 200, 256])
@pytest.mark.parametrize("dist", [gen.DIST_UNIFORM, gen.DIST_SKEW, gen.DIST_BINOMIAL])
def test_tile_boundaries_and_distributions(n, m, dist):
    ob, pb, gk = bucket_pair("delta", m)
    keys = gen.keys(n, seed=n, dist=dist, alpha=0.1, **gk)
    check_multisplit(keys, gen.values(n, seed=3), ob, pb)


@pytest.mark.parametrize("m", [2, 17, 256])
def test_single_bucket_is_copy(m):
    ob, pb, gk = bucket_pair("identity", m)
    n = 5 * T + 123
    keys = gen.keys(n, seed=4, dist=gen.DIST_SKEW, alpha=0.0, **gk)
    vals = gen.values(n, seed=4, parity=False)
    ko, vo, off = ms.multisplit(dev(keys), dev(vals), bucket=pb)
    assert np.array_equal(host(ko), keys) and np.array_equal(host(vo), vals)
    check_multisplit(keys, vals, ob, pb)


@pytest.mark.parametrize("kind", ["delta", "identity", "radix"])
def test_unaligned_inputs(kind):
    # inputs not 16-byte aligned take the non-TMA load path
    ob, pb, gk = bucket_pair(kind, 37)
    n = 3 * T + 11
    keys = gen.keys(n + 1, seed=5, **gk)
    vals = gen.values(n + 1, seed=5)
    kd, vd = dev(keys), dev(vals)
    ko, vo, off = ms.multisplit(kd[1:], vd[1:], bucket=pb)
    ek, ev, eo = oracle.multisplit(keys[1:], ob, vals[1:])
    assert np.array_equal(host(ko), ek) and np.array_equal(host(vo), ev)
    assert np.array_equal(host(off), eo)


@pytest.mark.parametrize("m", [2, 37, 64])
def test_unaligned_outputs(m):
    # outputs not 16-byte aligned disable the whole-run TMA stores
    ob, pb, gk = bucket_pair("delta", m)
    n = 5 * T + 19
    keys = gen.keys(n, seed=8, dist=gen.DIST_SKEW, **gk)
    vals = gen.values(n, seed=8)
    ko = torch.empty(n + 3, dtype=torch.int32, device="cuda")[3:]
    vo = torch.empty(n + 1, dtype=torch.int32, device="cuda")[1:]
    ms.multisplit(dev(keys), dev(vals), bucket=pb, out_keys=ko, out_values=vo)
    ek, ev, _ = oracle.multisplit(keys, ob, vals)
    assert np.array_equal(host(ko), ek) and np.array_equal(host(vo), ev)


@pytest.fixture
def option():
    """Set libms options for one test and restore the defaults afterwards."""
    lib = ms._lib
    saved = {o: ms.get_option(o) for o in (lib.MS_OPT_RANK, lib.MS_OPT_RUN_STORES, lib.MS_OPT_PIPELINE,
                                           lib.MS_OPT_SORT)}
    yield ms.set_option
    for o, v in saved.items():
        ms.set_option(o, v)


def test_per_element_store_path(option):
    option(ms._lib.MS_OPT_RUN_STORES, 0)
    for m in (2, 32):
        ob, pb, gk = bucket_pair("delta", m)
        n = 7 * T + 5
        keys = gen.keys(n, seed=m, dist=gen.DIST_BINOMIAL, **gk)
        check_multisplit(keys, gen.values(n, seed=1), ob, pb)
        check_multisplit(keys, None, ob, pb)


@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("m", [3, 16, 32, 64, 128, 256])
def test_deterministic_rank_mode(option, m, pairs):
    """MS_RANK_PEER_MASKS (no reliance on reading R23) gives the same bit-exact result."""
    option(ms._lib.MS_OPT_RANK, ms._lib.MS_RANK_PEER_MASKS)
    ob, pb, gk = bucket_pair("delta", m)
    for n, dist in ((5 * T + 77, gen.DIST_UNIFORM), (3 * T + 1, gen.DIST_SKEW)):
        keys = gen.keys(n, seed=m + n, dist=dist, **gk)
        check_multisplit(keys, gen.values(n, seed=4) if pairs else None, ob, pb)


@pytest.mark.parametrize("pairs", [False, True])
def test_unaligned_inputs_many_tiles_producer_warp(pairs):
    """Unaligned input (no TMA loads) with aligned outputs, m <= 16 (producer-warp
    run stores), enough tiles per CTA range to lap the three-stage ring, ragged tail
    (the producer/consumer stage hand-off for non-TMA tiles)."""
    for m in (4, 16):
        ob, pb, gk = bucket_pair("delta", m)
        n = (1 << 24) + 4099
        keys = gen.keys(n + 1, seed=m, **gk)
        vals = gen.values(n + 1, seed=m) if pairs else None
        kd = dev(keys)[1:]
        vd = dev(vals)[1:] if pairs else None
        ko, vo, off = ms.multisplit(kd, vd, bucket=pb)
        ek, ev, eo = oracle.multisplit(keys[1:], ob, vals[1:] if pairs else None)
        assert np.array_equal(host(ko), ek)
        if pairs:
            assert np.array_equal(host(vo), ev)
        assert np.array_equal(host(off), eo)


def test_c1_exact():
    """BASELINE configs[0]: n = 2^10 uniform keys, m = 2 delta buckets (single-CTA path)."""
    ob, pb, gk = bucket_pair("delta", 2)
    for seed in (1, 2, 3):
        keys = gen.keys(1 << 10, seed=seed, **gk)
        check_multisplit(keys, None, ob, pb)
        check_multisplit(keys, gen.values(1 << 10, seed=seed), ob, pb)


@pytest.mark.parametrize("m", [2, 4, 8, 16, 32, 64, 128, 256])
@pytest.mark.parametrize("pairs", [False, True])
def test_sweep_m_multi_tile(m, pairs):
    """Every m of the bench sweep (delta buckets, Delta = ceil(2^32/m)) over many tiles."""
    ob, pb, gk = bucket_pair("delta", m)
    n = 37 * T + 1234
    keys = gen.keys(n, seed=100 + m, **gk)
    check_multisplit(keys, gen.values(n, seed=m) if pairs else None, ob, pb)


@pytest.mark.parametrize("m", [64, 128, 256])
@pytest.mark.parametrize("dist", [gen.DIST_UNIFORM, gen.DIST_SKEW])
def test_c3_radix_and_identity(m, dist):
    """configs[2] bucket kinds (identity, radix digit) at m = 64/128/256, uniform and 90 % skew."""
    for kind in ("identity", "radix"):
        ob, pb, gk = bucket_pair(kind, m)
        if kind == "radix":  # the bench's C3 radix digit: the low bits
            bits = m.bit_length() - 1
            ob, pb, gk = oracle.radix(0, bits), ms.Radix(0, bits), dict(kind=gen.RADIX, m=m, shift=0, bits=bits)
        n = 45 * 4096 + 3
        keys = gen.keys(n, seed=m, dist=dist, alpha=0.1, **gk)
        check_multisplit(keys, gen.values(n, seed=5), ob, pb)


def test_custom_delta_widths():
    for m, d in ((7, 1), (7, 3), (100, 12345), (256, 2**24 + 7), (3, 2**31 + 1)):
        ob, pb = oracle.delta(m, d), ms.Delta(m, d)
        keys = gen.keys(3 * T + 1, seed=d % 1000)
        keys[:64] = np.array([0, 1, d - 1, d, d + 1, m * d - 1, m * d, 0xFFFFFFFF] * 8, np.uint64).astype(np.uint32)
        check_multisplit(keys, gen.values(keys.size, seed=1), ob, pb)


@pytest.mark.parametrize("n", [100, 3 * T + 7])
def test_identity_domain_error_flag(n):
    keys = gen.keys(n, seed=6, kind=gen.IDENTITY, m=8)
    _, _, _ = ms.multisplit(dev(keys), bucket=ms.Identity(8))
    assert ms.device_status() == 0
    keys[n // 2] = 8
    ko, _, _ = ms.multisplit(dev(keys), bucket=ms.Identity(8))
    assert ms.device_status() == 5  # MS_ERR_KEY_DOMAIN
    ms.multisplit(dev(keys % 8), bucket=ms.Identity(8))
    assert ms.device_status() == 0  # the flag belongs to the most recent call


# ------------------------------------------------------------------ stages (H, G)

@pytest.mark.parametrize("m", [1, 2, 8, 33, 256])
@pytest.mark.parametrize("n", [1, T, 5 * T + 77])
def test_stage_prescan(m, n):
    ob, pb, gk = bucket_pair("delta", m)
    keys = gen.keys(n, seed=7, dist=gen.DIST_BINOMIAL, **gk)
    for tile in (T, T // 2, 1000, 37):
        H = ms.prescan(dev(keys), pb, tile=tile)
        assert np.array_equal(host(H), oracle.tile_histogram(keys, ob, tile))


@pytest.mark.parametrize("shape", [(1, 1), (1, 256), (4096, 2), (4096, 32), (2049, 33), (32768, 256), (5, 255)])
def test_stage_scan(shape):
    L, m = shape
    rng = np.random.default_rng(L * m)
    Hn = rng.integers(0, 60, shape, dtype=np.uint64).astype(np.uint32)
    G, off = ms.scan(dev(Hn))
    eG = oracle.global_scan(Hn)
    assert np.array_equal(host(G), eG)
    tot = Hn.astype(np.int64).sum(axis=0)
    assert np.array_equal(host(off).astype(np.int64), np.concatenate([[0], np.cumsum(tot)]))


# ------------------------------------------------------------------ radix sort (Sec.7.1)

@pytest.mark.parametrize("n", [0, 1, 1000, T, 4 * T + 9, 1 << 20])
@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("r", [0, 8])
def test_radix_sort(n, pairs, r):
    """r = 8: the benched configs[3] schedule, 4 x 8-bit passes over [0, 32); r = 0: the default."""
    keys = gen.keys(n, seed=9)
    keys[::5] &= np.uint32(0xFF00FF)  # duplicates make stability visible
    vals = gen.values(n, seed=9)
    ek, ev = oracle.radix_sort(keys, vals if pairs else None)
    ko, vo = ms.radix_sort(dev(keys), dev(vals) if pairs else None, begin_bit=0, end_bit=32, bits_per_pass=r)
    assert np.array_equal(host(ko), ek)
    if pairs:
        assert np.array_equal(host(vo), ev)


@pytest.mark.parametrize("args", [(0, 32, 4), (0, 32, 7), (0, 32, 5), (8, 24, 8), (3, 17, 6), (31, 32, 1)])
def test_radix_sort_bits(args):
    b0, b1, r = args
    n = 3 * T + 100
    keys = gen.keys(n, seed=b1)
    vals = gen.values(n, seed=1)
    ek, ev = oracle.radix_sort(keys, vals, b0, b1)
    ko, vo = ms.radix_sort(dev(keys), dev(vals), begin_bit=b0, end_bit=b1, bits_per_pass=r)
    assert np.array_equal(host(ko), ek) and np.array_equal(host(vo), ev)


@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("m", [2, 37, 256])
def test_three_launch_mode(option, pairs, m):
    # MS_PIPELINE_TILE: the paper's {tile histograms H, scan of H, postscan}
    option(ms._lib.MS_OPT_PIPELINE, ms._lib.MS_PIPELINE_TILE)
    ob, pb, gk = bucket_pair("delta", m)
    n = 29 * T + 333
    keys = gen.keys(n, seed=m, dist=gen.DIST_SKEW, **gk)
    check_multisplit(keys, gen.values(n, seed=2) if pairs else None, ob, pb)


def test_determinism_repeated_runs():
    n, m = 40 * T + 17, 64
    ob, pb, gk = bucket_pair("delta", m)
    keys = dev(gen.keys(n, seed=10, dist=gen.DIST_SKEW, **gk))
    vals = dev(gen.values(n, seed=10))
    ref = ms.multisplit(keys, vals, bucket=pb)
    for _ in range(20):
        out = ms.multisplit(keys, vals, bucket=pb)
        for a, b in zip(ref, out):
            assert torch.equal(a, b)
