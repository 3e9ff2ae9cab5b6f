"""Sharded multisplit on one GPU.

* The fused path KP (ms_shard_prescan -> gathered counts -> ms_shard_scatter,
  Eq.3 with the GPUs as level 0) with G virtual ranks: every rank's
  kernels store straight into the other ranks' output shards; the all-gather
  becomes the shared count matrix.  The concatenation of the output shards
  must equal the oracle's stable multisplit of the concatenated input.
* The library's own sharded call (NCCL inside libms) at world_size 1 through
  both paths: registered output windows (KP) and unregistered outputs (NCCL
  send/receive + KX merge).
* The KX merge kernel under the NCCL path's plan with virtual ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
from gen import inputs as gen

pytestmark = pytest.mark.gpu
ms = pytest.importorskip("paper_1701_01189_b200")
from paper_1701_01189_b200 import sharded  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint32)


def split(keys, vals, sizes):
    b = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ks = [_dev(keys[b[r]:b[r + 1]]) for r in range(len(sizes))]
    vs = [_dev(vals[b[r]:b[r + 1]]) for r in range(len(sizes))] if vals is not None else None
    return ks, vs


@pytest.mark.parametrize("sizes", [[70000], [40000, 40000], [100003, 3, 50000], [30000] * 8,
                                   [0, 65536, 8193, 1, 77777]])
@pytest.mark.parametrize("m", [2, 16, 33, 256])
@pytest.mark.parametrize("pairs", [False, True])
def test_fused_kp_virtual_ranks(sizes, m, pairs):
    ms.device_init(0)
    n = sum(sizes)
    ob = oracle.delta(m)
    keys = gen.keys(n, seed=n + m, kind=gen.DELTA, m=m, delta=ob.delta, dist=gen.DIST_SKEW, alpha=0.4)
    vals = gen.values(n, seed=1) if pairs else None
    ks, vs = split(keys, vals, sizes)
    ok, ov, goff = sharded.virtual_ranks(ks, vs, ms.Delta(m))
    ek, ev, eo = oracle.multisplit(keys, ob, vals)
    assert [x.numel() for x in ok] == sizes
    assert np.array_equal(np.concatenate([_host(x) for x in ok]), ek)
    if pairs:
        assert np.array_equal(np.concatenate([_host(x) for x in ov]), ev)
    assert goff.cpu().numpy().tolist() == eo.astype(np.int64).tolist()


def test_fused_kp_identity_radix():
    ms.device_init(0)
    sizes = [50000, 12345, 99999]
    n = sum(sizes)
    for bucket, ob, gk in ((ms.Identity(64), oracle.identity(64), dict(kind=gen.IDENTITY, m=64)),
                           (ms.Radix(8, 8), oracle.radix(8, 8), dict(kind=gen.RADIX, m=256, shift=8, bits=8))):
        keys = gen.keys(n, seed=5, **gk)
        ks, _ = split(keys, None, sizes)
        ok, _, _ = sharded.virtual_ranks(ks, None, bucket)
        ek, _, _ = oracle.multisplit(keys, ob)
        assert np.array_equal(np.concatenate([_host(x) for x in ok]), ek)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def comm1():
    """A world_size-1 process group (gloo for the id broadcast) and an ms_comm over it."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    c = sharded.Comm()
    yield c
    c.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [2, 32, 64, 256])
@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("registered", [False, True])
def test_sharded_call_world1(comm1, m, pairs, registered):
    ms.device_init(0)
    n = 3 * 8192 + 1234
    ob = oracle.delta(m)
    keys = gen.keys(n, seed=m, kind=gen.DELTA, m=m, delta=ob.delta, dist=gen.DIST_SKEW, alpha=0.3)
    vals = gen.values(n, seed=2) if pairs else None
    ko = torch.empty(n, dtype=torch.int32, device="cuda")
    vo = torch.empty(n, dtype=torch.int32, device="cuda") if pairs else None
    if registered:
        comm1.register_output(ko, vo)
    else:
        comm1.register_output(torch.empty(1, dtype=torch.int32, device="cuda"))  # other windows
    rk, rv, goff = sharded.multisplit(comm1, _dev(keys), _dev(vals) if pairs else None, bucket=ms.Delta(m),
                                      out_keys=ko, out_values=vo)
    ek, ev, eo = oracle.multisplit(keys, ob, vals)
    assert np.array_equal(_host(rk), ek)
    if pairs:
        assert np.array_equal(_host(rv), ev)
    assert goff.cpu().numpy().tolist() == eo.astype(np.int64).tolist()


def test_comm_failure_detection_world1():
    """ms_comm_check on a healthy communicator, then ms_comm_abort + close (a fresh comm:
    the module fixture keeps its own)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        c = sharded.Comm()
        c.check()
        c.abort()
        c.close()
    finally:
        if own:
            dist.destroy_process_group()


def run_merge_virtual(keys_np, vals_np, sizes, bucket):
    """The NCCL path's plan + KX merge with the send/receive done by slicing."""
    G = len(sizes)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    locals_ = []
    for r in range(G):
        k = _dev(keys_np[bounds[r]:bounds[r + 1]])
        v = None if vals_np is None else _dev(vals_np[bounds[r]:bounds[r + 1]])
        locals_.append(ms.multisplit(k, v, bucket=bucket))
    C = np.stack([(off[1:].to(torch.int64) - off[:-1].to(torch.int64)).cpu().numpy() for _, _, off in locals_])
    plans = [sharded.shard_plan(C.astype(np.uint64), r) for r in range(G)]
    lib = ms._lib.load()
    import ctypes
    outs_k, outs_v = [], []
    for r in range(G):
        sl = lambda t, s: t[int(plans[s]["send_displs"][r]):int(plans[s]["send_displs"][r] + plans[s]["send_counts"][r])]  # noqa: E731
        rk = torch.cat([sl(locals_[s][0], s) for s in range(G)])
        rv = torch.cat([sl(locals_[s][1], s) for s in range(G)]) if vals_np is not None else None
        starts = _dev(np.append(plans[r]["recv_displs"], rk.numel()).astype(np.uint32))
        offs = _dev(plans[r]["merge_offsets"])
        ko = torch.empty_like(rk)
        fn = bucket.c()
        if rv is not None:
            vo = torch.empty_like(rv)
            ms._lib.check(lib.ms_shard_merge_pairs(rk.data_ptr(), rv.data_ptr(), rk.numel(), ctypes.byref(fn),
                                                   starts.data_ptr(), offs.data_ptr(), G, ko.data_ptr(),
                                                   vo.data_ptr(), None))
            outs_v.append(_host(vo))
        else:
            ms._lib.check(lib.ms_shard_merge_keys(rk.data_ptr(), rk.numel(), ctypes.byref(fn), starts.data_ptr(),
                                                  offs.data_ptr(), G, ko.data_ptr(), None))
        outs_k.append(_host(ko))
    return outs_k, outs_v, plans[0]["global_offsets"]


@pytest.mark.parametrize("sizes", [[40000, 40000], [100003, 3, 50000], [0, 65536, 8193, 1, 77777]])
@pytest.mark.parametrize("m", [2, 33, 256])
def test_merge_path_virtual_ranks(sizes, m):
    n = sum(sizes)
    ob = oracle.delta(m)
    keys = gen.keys(n, seed=n + m, kind=gen.DELTA, m=m, delta=ob.delta, dist=gen.DIST_SKEW, alpha=0.4)
    vals = gen.values(n, seed=1)
    ok, ov, goff = run_merge_virtual(keys, vals, sizes, ms.Delta(m))
    ek, ev, eo = oracle.multisplit(keys, ob, vals)
    assert np.array_equal(np.concatenate(ok), ek) and np.array_equal(np.concatenate(ov), ev)
    assert goff.astype(np.int64).tolist() == eo.astype(np.int64).tolist()
