"""GPU parity of the one-pass pipeline (csrc/ms_onesweep.cuh)
against the CPU oracle, element by element, bit-exact.

- the radix sort's default path (MS_SORT_AUTO): every digit histogram in one
  read (KOH), then one fused rank / decoupled look-back / scatter pass (KO)
  per digit -- schedules of 1..8 passes, ragged tails around the KO tile
  (12288 keys, 8192 pairs), duplicated and skewed keys (the hot-digit ballot
  path), unaligned inputs (the non-TMA loads), repeated calls;
- the one-pass multisplit (MS_PIPELINE_ONESWEEP) over the SPEC m grid and the
  four bucket identifiers, keys and pairs, uniform / skewed / single-bucket,
  the identity domain-error flag;
- both against the paper-faithful per-pass path (MS_SORT_PASSES).
"""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gen

pytestmark = pytest.mark.gpu

ms = pytest.importorskip("paper_1701_01189_b200")
TK, TP = 12288, 8192  # KO tiles: keys (24 compute warps x 512), pairs (16 x 512)


def dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


@pytest.fixture
def option():
    lib = ms._lib
    saved = {o: ms.get_option(o) for o in (lib.MS_OPT_RANK, lib.MS_OPT_PIPELINE, lib.MS_OPT_SORT)}
    yield ms.set_option
    for o, v in saved.items():
        ms.set_option(o, v)


def test_sort_default_is_onesweep():
    assert ms.get_option(ms._lib.MS_OPT_SORT) == ms._lib.MS_SORT_AUTO


def check_sort(keys, vals, b0=0, b1=32, r=8):
    ek, ev = oracle.radix_sort(keys, vals, b0, b1)
    ko, vo = ms.radix_sort(dev(keys), None if vals is None else dev(vals), begin_bit=b0, end_bit=b1,
                           bits_per_pass=r)
    assert np.array_equal(host(ko), ek), "keys differ"
    if vals is not None:
        assert np.array_equal(host(vo), ev), "values differ"


SIZES = [1, 2, 33, TP - 1, TP, TP + 1, TK - 1, TK, TK + 1, 3 * TK + 7, 37 * TK + 4095]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("pairs", [False, True])
def test_sort_sizes(n, pairs):
    keys = gen.keys(n, seed=n)
    keys[::3] &= np.uint32(0x00FF00FF)  # duplicates: stability visible
    check_sort(keys, gen.values(n, seed=n) if pairs else None)


@pytest.mark.parametrize("args", [(0, 32, 8), (0, 32, 4), (0, 32, 5), (0, 32, 6), (0, 32, 7), (0, 28, 7), (4, 32, 7), (8, 24, 8),
                                  (3, 17, 6), (31, 32, 1), (0, 8, 8), (0, 16, 8), (5, 29, 3), (0, 32, 0)])
@pytest.mark.parametrize("pairs", [False, True])
def test_sort_schedules(args, pairs):
    b0, b1, r = args
    n = 9 * TK + 333
    keys = gen.keys(n, seed=b1 + r)
    check_sort(keys, gen.values(n, seed=2) if pairs else None, b0, b1, r)


@pytest.mark.parametrize("pattern", ["small", "constant", "two", "hot90", "sorted", "reversed", "topzero"])
@pytest.mark.parametrize("pairs", [False, True])
def test_sort_key_patterns(pattern, pairs):
    """Skewed digits: one digit value holding most keys takes the hot-bucket ballot rank."""
    n = 21 * TK + 5
    keys = gen.keys(n, seed=17)
    if pattern == "small":
        keys &= np.uint32(0xFF)           # three of four digits constant
    elif pattern == "constant":
        keys[:] = np.uint32(0xDEADBEEF)
    elif pattern == "two":
        keys = np.where(keys & 1, np.uint32(7), np.uint32(0xFFFFFFF0)).astype(np.uint32)
    elif pattern == "hot90":
        hot = (gen.keys(n, seed=18) % np.uint32(10)) != 0
        keys[hot] = np.uint32(0x12345678)
    elif pattern == "sorted":
        keys = np.sort(keys)
    elif pattern == "reversed":
        keys = np.sort(keys)[::-1].copy()
    elif pattern == "topzero":
        keys >>= np.uint32(8)
    check_sort(keys, gen.values(n, seed=19) if pairs else None)


@pytest.mark.parametrize("pairs", [False, True])
def test_sort_unaligned_inputs(pairs):
    n = 5 * TK + 13
    keys = gen.keys(n + 1, seed=23)
    vals = gen.values(n + 1, seed=23)
    ek, ev = oracle.radix_sort(keys[1:], vals[1:] if pairs else None)
    kd, vd = dev(keys), dev(vals)
    ko, vo = ms.radix_sort(kd[1:], vd[1:] if pairs else None, bits_per_pass=8)
    assert np.array_equal(host(ko), ek)
    if pairs:
        assert np.array_equal(host(vo), ev)


@pytest.mark.parametrize("pairs", [False, True])
def test_sort_matches_per_pass_path(option, pairs):
    n = 50 * TK + 999
    keys = dev(gen.keys(n, seed=29))
    vals = dev(gen.values(n, seed=29)) if pairs else None
    a = ms.radix_sort(keys, vals, bits_per_pass=8)
    option(ms._lib.MS_OPT_SORT, ms._lib.MS_SORT_PASSES)
    b = ms.radix_sort(keys, vals, bits_per_pass=8)
    assert torch.equal(a[0], b[0])
    if pairs:
        assert torch.equal(a[1], b[1])


def test_sort_repeated_recycled_workspace():
    n = 30 * TK + 1
    keys = dev(gen.keys(n, seed=31))
    vals = dev(gen.values(n, seed=31))
    ws = torch.empty(ms.radix_sort_workspace_size(n, True), dtype=torch.uint8, device="cuda")
    ref = ms.radix_sort(keys, vals, workspace=ws)
    for i in range(10):
        ws.fill_(0xA5 if i % 2 else 0x00)
        out = ms.radix_sort(keys, vals, workspace=ws)
        assert torch.equal(ref[0], out[0]) and torch.equal(ref[1], out[1])


# ------------------------------------------------------------------ one-pass multisplit

def bucket_pair(kind: str, m: int):
    if kind == "delta":
        o = oracle.delta(m)
        return o, ms.Delta(m), dict(kind=gen.DELTA, m=m, delta=o.delta)
    if kind == "identity":
        return oracle.identity(m), ms.Identity(m), dict(kind=gen.IDENTITY, m=m)
    if kind == "splitters":
        rng = np.random.default_rng(m)
        spl = np.unique(rng.integers(1, 1 << 32, size=m - 1, dtype=np.uint64).astype(np.uint32))
        while spl.size < m - 1:
            spl = np.unique(np.concatenate([spl, rng.integers(1, 1 << 32, size=m, dtype=np.uint64).astype(np.uint32)]))[:m - 1]
        return oracle.splitters(spl), ms.Splitters(dev(spl)), dict(kind=gen.DELTA, m=m, delta=oracle.delta(m).delta)
    bits = max(1, (m - 1).bit_length())
    shift = 32 - bits - 3
    return oracle.radix(shift, bits), ms.Radix(shift, bits), dict(kind=gen.RADIX, m=1 << bits, shift=shift,
                                                                     bits=bits)


def check_multisplit(keys, vals, ob, pb):
    ek, ev, eo = oracle.multisplit(keys, ob, vals)
    ko, vo, off = ms.multisplit(dev(keys), None if vals is None else dev(vals), bucket=pb)
    assert np.array_equal(host(ko), ek), "keys differ"
    if vals is not None:
        assert np.array_equal(host(vo), ev), "values differ"
    assert np.array_equal(host(off), eo), "bucket offsets differ"
    assert ms.device_status() == 0


@pytest.mark.parametrize("m", [1, 2, 3, 8, 32, 33, 64, 255, 256])
@pytest.mark.parametrize("kind", ["delta", "identity", "radix", "splitters"])
@pytest.mark.parametrize("pairs", [False, True])
def test_onesweep_multisplit_grid(option, m, kind, pairs):
    if kind == "radix" and m == 1:
        pytest.skip("radix digits have m = 2^bits >= 2")
    option(ms._lib.MS_OPT_PIPELINE, ms._lib.MS_PIPELINE_ONESWEEP)
    ob, pb, gk = bucket_pair(kind, m)
    for n, dist in ((7 * TK + 77, gen.DIST_UNIFORM), (5000, gen.DIST_UNIFORM), (3 * TK + 1, gen.DIST_SKEW)):
        keys = gen.keys(n, seed=m + n, dist=dist, **gk)
        check_multisplit(keys, gen.values(n, seed=4) if pairs else None, ob, pb)


@pytest.mark.parametrize("m", [2, 64, 256])
def test_onesweep_single_bucket_and_domain_error(option, m):
    option(ms._lib.MS_OPT_PIPELINE, ms._lib.MS_PIPELINE_ONESWEEP)
    ob, pb, gk = bucket_pair("identity", m)
    n = 6 * TK + 3
    keys = gen.keys(n, seed=5, dist=gen.DIST_SKEW, alpha=0.0, **gk)
    check_multisplit(keys, gen.values(n, seed=5), ob, pb)
    keys[n // 2] = np.uint32(m + 5)  # identity key >= m: sticky flag
    kd = dev(keys)
    ms.multisplit(kd, None, bucket=pb)
    assert ms.device_status() == ms._lib.MS_ERR_KEY_DOMAIN


@pytest.mark.parametrize("pipe", ["AUTO", "LEVEL0"])
@pytest.mark.parametrize("m", [128, 129, 200, 256])
@pytest.mark.parametrize("dist", [gen.DIST_UNIFORM, gen.DIST_SKEW])
def test_pairs_wide_m_default_and_level0(option, pipe, m, dist):
    """AUTO sends pairs with m > 128 through the one-pass pipeline; LEVEL0 keeps KMW -> KFW."""
    option(ms._lib.MS_OPT_PIPELINE, getattr(ms._lib, "MS_PIPELINE_" + pipe))
    ob, pb, gk = bucket_pair("identity", m)
    n = 11 * TP + 517
    keys = gen.keys(n, seed=m + 3, dist=dist, alpha=0.1, **gk)
    check_multisplit(keys, gen.values(n, seed=m), ob, pb)


@pytest.mark.parametrize("pairs", [False, True])
def test_sort_many_tiles_per_cta(pairs):
    """Past 148 tiles per launch: every persistent CTA takes several tiles (ticket order,
    deferred scatter, stage reuse, look-back across CTAs), element by element."""
    n = 148 * 3 * TK + 4099
    keys = gen.keys(n, seed=41)
    keys[::7] &= np.uint32(0xFFFF00FF)
    check_sort(keys, gen.values(n, seed=41) if pairs else None)


@pytest.mark.parametrize("what", ["sort_keys", "sort_pairs", "ms_pairs_256"])
def test_one_pass_in_cuda_graph(what):
    """The one-pass pipeline captured in a CUDA graph and replayed on new inputs: the
    memset node re-zeroes the tickets and look-back words on every replay."""
    n = 20 * TK + 11
    pairs = what != "sort_keys"
    ks = torch.empty(n, dtype=torch.int32, device="cuda")
    vs = torch.empty(n, dtype=torch.int32, device="cuda") if pairs else None
    ko = torch.empty_like(ks)
    vo = torch.empty_like(vs) if pairs else None
    gk = {}
    if what == "ms_pairs_256":
        ob, pb, gk = bucket_pair("identity", 256)
        off = torch.empty(257, dtype=torch.int32, device="cuda")
        ws = torch.empty(ms.workspace_size(n, 256, True), dtype=torch.uint8, device="cuda")
        call = lambda: ms.multisplit(ks, vs, bucket=pb, out_keys=ko, out_values=vo,  # noqa: E731
                                     out_offsets=off, workspace=ws)
    else:
        ws = torch.empty(ms.radix_sort_workspace_size(n, pairs), dtype=torch.uint8, device="cuda")
        call = lambda: ms.radix_sort(ks, vs, bits_per_pass=8, out_keys=ko, out_values=vo,  # noqa: E731
                                     workspace=ws)
    ms.device_init(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside the capture (kernel attributes)
        ks.copy_(dev(gen.keys(n, seed=1, **gk)))
        if pairs:
            vs.copy_(dev(gen.values(n, seed=1)))
        call()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        call()
    for seed in (2, 3, 4):
        kh = gen.keys(n, seed=seed, **gk)
        vh = gen.values(n, seed=seed) if pairs else None
        ks.copy_(dev(kh))
        if pairs:
            vs.copy_(dev(vh))
        g.replay()
        torch.cuda.synchronize()
        if what == "ms_pairs_256":
            ek, ev, eo = oracle.multisplit(kh, ob, vh)
            assert np.array_equal(host(off), eo)
        else:
            ek, ev = oracle.radix_sort(kh, vh)
        assert np.array_equal(host(ko), ek)
        if pairs:
            assert np.array_equal(host(vo), ev)
