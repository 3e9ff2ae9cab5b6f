"""CPU-side tests of the C ABI: libms.so loads without a GPU, exports every
symbol include/multisplit.h declares, and its host-only logic (argument
validation, workspace sizing, bucket helpers, radix pass schedule) behaves as
documented.  No compute call is made here."""
import ctypes
import os
import re

import pytest

from paper_1701_01189_b200 import _lib
from tests.conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "multisplit.h")


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ms_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), f"libms.so does not export {name}"
    bound = {s[0] for s in _lib.SIGNATURES}
    assert bound == set(names), "binding signatures out of sync with the header"


def test_status_strings_and_version(lib):
    assert lib.ms_status_string(0) == b"MS_SUCCESS"
    assert lib.ms_status_string(5) == b"MS_ERR_KEY_DOMAIN"
    assert lib.ms_version().decode().count(".") == 2


def test_radix_schedule_golden(lib):
    # SPEC S:322 / P:1716
    for ln in golden("spec_s322_radix_schedule.txt"):
        r, rest = ln.split(":")
        r = int(r.strip()[2:])
        import paper_1701_01189_b200 as ms
        sched = ms.radix_pass_schedule(0, 32, r)
        assert [b for _, b in sched] == [int(x) for x in rest.split()]
        assert [s for s, _ in sched] == [r * i for i in range(len(sched))]
    assert lib.ms_radix_pass_schedule(0, 32, 9, None, None, 0) == -1
    assert lib.ms_radix_pass_schedule(8, 8, 4, None, None, 0) == -1
    assert lib.ms_radix_pass_schedule(4, 20, 8, None, None, 0) == 2
    # bits_per_pass = 0: the library's choice, 8-bit digits (four passes)
    import paper_1701_01189_b200 as ms
    assert ms.radix_pass_schedule(0, 32, 0) == ms.radix_pass_schedule(0, 32, 8)
    assert [b for _, b in ms.radix_pass_schedule(0, 32, 0)] == [8, 8, 8, 8]


def test_bucket_helpers(lib):
    fn = _lib.ms_bucket_fn()
    for m in (1, 2, 3, 255, 256):
        assert lib.ms_bucket_delta_default(m, ctypes.byref(fn)) == 0
        assert fn.kind == _lib.MS_BUCKET_DELTA and fn.num_buckets == m
        assert fn.delta == min(-(-(1 << 32) // m), (1 << 32) - 1)
    assert lib.ms_bucket_delta_default(0, ctypes.byref(fn)) == _lib.MS_ERR_UNSUPPORTED
    # m > 256 (Sec.6.3): up to 65536 buckets through the multisplit entry points
    assert lib.ms_bucket_delta_default(257, ctypes.byref(fn)) == 0 and fn.delta == -(-(1 << 32) // 257)
    assert lib.ms_bucket_delta_default(65537, ctypes.byref(fn)) == _lib.MS_ERR_UNSUPPORTED
    assert lib.ms_bucket_radix(8, 16, ctypes.byref(fn)) == 0 and fn.num_buckets == 65536
    assert lib.ms_bucket_radix(0, 17, ctypes.byref(fn)) == _lib.MS_ERR_INVALID_VALUE
    spl = _lib.ms_bucket_fn(_lib.MS_BUCKET_SPLITTERS, 4, 0, 0, 0, None)
    assert lib.ms_bucket_validate(ctypes.byref(spl)) == _lib.MS_ERR_INVALID_VALUE  # no table
    one = _lib.ms_bucket_fn(_lib.MS_BUCKET_SPLITTERS, 1, 0, 0, 0, None)
    assert lib.ms_bucket_validate(ctypes.byref(one)) == 0
    assert lib.ms_bucket_radix(24, 8, ctypes.byref(fn)) == 0 and fn.num_buckets == 256
    assert lib.ms_bucket_radix(25, 8, ctypes.byref(fn)) == _lib.MS_ERR_INVALID_VALUE
    assert lib.ms_bucket_radix(0, 0, ctypes.byref(fn)) == _lib.MS_ERR_INVALID_VALUE
    bad = _lib.ms_bucket_fn(_lib.MS_BUCKET_RADIX, 128, 0, 0, 8)
    assert lib.ms_bucket_validate(ctypes.byref(bad)) == _lib.MS_ERR_INVALID_VALUE
    bad = _lib.ms_bucket_fn(_lib.MS_BUCKET_DELTA, 4, 0, 0, 0)
    assert lib.ms_bucket_validate(ctypes.byref(bad)) == _lib.MS_ERR_INVALID_VALUE
    bad = _lib.ms_bucket_fn(7, 4, 1, 0, 0)
    assert lib.ms_bucket_validate(ctypes.byref(bad)) == _lib.MS_ERR_INVALID_VALUE


def test_host_argument_errors_return_before_launch(lib):
    # These return from host validation; nothing touches the (absent) GPU.
    fn = _lib.ms_bucket_fn(_lib.MS_BUCKET_DELTA, 0, 1, 0, 0)
    fake = ctypes.c_void_p(0x10000)
    other = ctypes.c_void_p(0x20000000)
    ws = ctypes.c_void_p(0x40000000)
    assert lib.ms_multisplit_keys(fake, other, 10, ctypes.byref(fn), None, ws, 1 << 20, None) == \
        _lib.MS_ERR_UNSUPPORTED
    fn = _lib.ms_bucket_fn(_lib.MS_BUCKET_DELTA, 4, 1 << 30, 0, 0)
    assert lib.ms_multisplit_keys(None, other, 10, ctypes.byref(fn), None, ws, 1 << 20, None) == \
        _lib.MS_ERR_INVALID_VALUE
    assert lib.ms_multisplit_keys(fake, fake, 10, ctypes.byref(fn), None, ws, 1 << 20, None) == \
        _lib.MS_ERR_INVALID_VALUE                                    # in-place is rejected
    assert lib.ms_multisplit_keys(fake, ctypes.c_void_p(0x10000 + 8), 10, ctypes.byref(fn), None, ws,
                                  1 << 20, None) == _lib.MS_ERR_INVALID_VALUE  # overlap
    assert lib.ms_multisplit_keys(fake, other, 10, ctypes.byref(fn), None, ws, 1, None) == \
        _lib.MS_ERR_WORKSPACE
    assert lib.ms_multisplit_keys(fake, other, 1 << 32, ctypes.byref(fn), None, ws, 1 << 40, None) == \
        _lib.MS_ERR_UNSUPPORTED
    assert lib.ms_multisplit_pairs(fake, None, other, None, 10, ctypes.byref(fn), None, ws, 1 << 20,
                                   None) == _lib.MS_ERR_INVALID_VALUE
    assert lib.ms_radix_sort_keys(fake, other, 10, 0, 32, 9, ws, 1 << 30, None) == _lib.MS_ERR_INVALID_VALUE
    assert lib.ms_radix_sort_keys(fake, other, 10, 0, 32, 8, ws, 10, None) == _lib.MS_ERR_WORKSPACE
    assert lib.ms_stage_prescan(fake, 10, ctypes.byref(fn), other, 0, None) == _lib.MS_ERR_INVALID_VALUE


def test_workspace_sizes(lib):
    T = lib.ms_multisplit_tile_size(256, 1)
    assert T >= 1024 and T & (T - 1) == 0
    small = lib.ms_multisplit_workspace_size(T, 256, 1)
    big = lib.ms_multisplit_workspace_size(T + 1, 256, 1)
    assert small < big
    n = 1 << 25
    L = -(-n // T)
    assert lib.ms_multisplit_workspace_size(n, 256, 1) >= L * 256 * 4    # holds H (m x L words)
    assert lib.ms_radix_sort_workspace_size(n, 1) >= 2 * 4 * n           # alternate keys + values
    assert lib.ms_radix_sort_workspace_size(n, 0) >= 4 * n


def test_no_cpu_fallback_in_product_path():
    # The binding must not import the oracle or numpy-based compute.
    import paper_1701_01189_b200 as ms
    src = open(ms.__file__).read() + open(_lib.__file__).read()
    assert "oracle" not in src.replace("no CPU fallback", "")


def test_options_host(lib):
    """ms_set_option / ms_get_option are host-only: defaults, validation, round trip."""
    assert lib.ms_get_option(_lib.MS_OPT_RANK) == _lib.MS_RANK_AUTO
    assert lib.ms_get_option(_lib.MS_OPT_RUN_STORES) == 1
    assert lib.ms_get_option(_lib.MS_OPT_PIPELINE) == _lib.MS_PIPELINE_AUTO
    assert lib.ms_get_option(_lib.MS_OPT_SORT) == _lib.MS_SORT_AUTO
    assert lib.ms_get_option(4) == -1
    assert lib.ms_set_option(_lib.MS_OPT_RANK, 5) == _lib.MS_ERR_INVALID_VALUE
    assert lib.ms_set_option(9, 0) == _lib.MS_ERR_INVALID_VALUE
    assert lib.ms_set_option(_lib.MS_OPT_RANK, _lib.MS_RANK_PEER_MASKS) == 0
    assert lib.ms_get_option(_lib.MS_OPT_RANK) == _lib.MS_RANK_PEER_MASKS
    assert lib.ms_set_option(_lib.MS_OPT_RANK, _lib.MS_RANK_AUTO) == 0
    for v in (_lib.MS_PIPELINE_LEVEL0, _lib.MS_PIPELINE_TILE, _lib.MS_PIPELINE_ONESWEEP, _lib.MS_PIPELINE_AUTO):
        assert lib.ms_set_option(_lib.MS_OPT_PIPELINE, v) == 0 and lib.ms_get_option(_lib.MS_OPT_PIPELINE) == v
    assert lib.ms_set_option(_lib.MS_OPT_PIPELINE, 4) == _lib.MS_ERR_INVALID_VALUE
    assert lib.ms_set_option(_lib.MS_OPT_SORT, _lib.MS_SORT_PASSES) == 0
    assert lib.ms_get_option(_lib.MS_OPT_SORT) == _lib.MS_SORT_PASSES
    assert lib.ms_set_option(_lib.MS_OPT_SORT, 2) == _lib.MS_ERR_INVALID_VALUE
    assert lib.ms_set_option(_lib.MS_OPT_SORT, _lib.MS_SORT_AUTO) == 0


def test_workspace_alignment_rejected(lib):
    """A workspace that is not 256-byte aligned is rejected before any launch."""
    fn = _lib.ms_bucket_fn(_lib.MS_BUCKET_DELTA, 4, 1 << 30, 0, 0)
    st = lib.ms_multisplit_keys(0x1000, 0x2000, 0, ctypes.byref(fn), None, 0x10010, 1 << 20, None)
    assert st == _lib.MS_ERR_INVALID_VALUE
    st = lib.ms_radix_sort_keys(0x1000, 0x2000, 10, 0, 32, 8, 0x10004, 1 << 30, None)
    assert st == _lib.MS_ERR_INVALID_VALUE
