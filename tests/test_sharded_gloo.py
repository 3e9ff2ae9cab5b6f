"""Host logic of the sharded multisplit on CPU: the plan
(ms_shard_plan, the C host code libms's NCCL path runs) checked for
consistency, and the exchange it drives (all-gather of counts, plan,
all-to-all-v, merge placement) run by world_size 2 and 3 gloo process groups
(sharded.exchange_reference).  The GPU steps (local multisplit, merge kernel)
are replaced here by stand-ins built on the oracle; the library's own sharded
calls (NCCL inside libms, fused KP scatter) are covered by
tests/test_gpu_sharded.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from gen import inputs as gen
from paper_1701_01189_b200 import sharded
from paper_1701_01189_b200 import Delta, Identity


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _to_oracle(bucket):
    if bucket.kind == 1:
        return oracle.delta(bucket.m, bucket.delta)
    if bucket.kind == 0:
        return oracle.identity(bucket.m)
    return oracle.radix(bucket.shift, bucket.bits)


def oracle_local(keys, values, bucket):
    k = keys.numpy().view(np.uint32)
    v = None if values is None else values.numpy().view(np.uint32)
    ko, vo, off = oracle.multisplit(k, _to_oracle(bucket), v)
    t = lambda a: None if a is None else torch.from_numpy(a.view(np.int32).copy())  # noqa: E731
    return t(ko), t(vo), torch.from_numpy(off.astype(np.int64))


def numpy_merge(keys_recv, vals_recv, bucket, recv_displs, merge_offsets, G):
    """Stand-in for ms_shard_merge_*: out[merge_offsets[s][f(key)] + e] = element e."""
    fn = _to_oracle(bucket)
    k = keys_recv.numpy().view(np.uint32)
    n = k.size
    starts = np.append(recv_displs.astype(np.int64), n)
    ko = np.empty(n, np.uint32)
    vo = np.empty(n, np.uint32) if vals_recv is not None else None
    for s in range(G):
        for e in range(int(starts[s]), int(starts[s + 1])):
            p = (int(merge_offsets[s, oracle.bucket_of(fn, int(k[e]))]) + e) & 0xFFFFFFFF
            ko[p] = k[e]
            if vo is not None:
                vo[p] = vals_recv.numpy().view(np.uint32)[e]
    t = lambda a: None if a is None else torch.from_numpy(a.view(np.int32).copy())  # noqa: E731
    return t(ko), t(vo)


def _worker(rank, world, port, sizes, m, kind, pairs, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = sum(sizes)
    bucket = Delta(m) if kind == "delta" else Identity(m)
    gk = dict(kind=gen.DELTA, m=m, delta=bucket.delta) if kind == "delta" else dict(kind=gen.IDENTITY, m=m)
    keys = gen.keys(n, seed=42, dist=gen.DIST_SKEW, alpha=0.3, **gk)
    vals = gen.values(n, seed=42)
    lo = sum(sizes[:rank])
    hi = lo + sizes[rank]
    k = torch.from_numpy(keys[lo:hi].view(np.int32).copy())
    v = torch.from_numpy(vals[lo:hi].view(np.int32).copy()) if pairs else None
    ko, vo, go = sharded.exchange_reference(k, v, bucket, oracle_local, numpy_merge)
    np.save(os.path.join(out_dir, f"k{rank}.npy"), ko.numpy().view(np.uint32))
    if pairs:
        np.save(os.path.join(out_dir, f"v{rank}.npy"), vo.numpy().view(np.uint32))
    np.save(os.path.join(out_dir, f"o{rank}.npy"), go)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sizes,m,kind,pairs", [
    ([700, 700], 4, "delta", True),
    ([1000, 13], 33, "delta", True),
    ([0, 500, 250], 7, "identity", False),
    ([333, 1, 666], 256, "delta", True),
])
def test_sharded_gloo(tmp_path, sizes, m, kind, pairs):
    world = len(sizes)
    port = _free_port()
    mp.spawn(_worker, args=(world, port, sizes, m, kind, pairs, str(tmp_path)), nprocs=world, join=True)
    n = sum(sizes)
    bucket = Delta(m) if kind == "delta" else Identity(m)
    gk = dict(kind=gen.DELTA, m=m, delta=bucket.delta) if kind == "delta" else dict(kind=gen.IDENTITY, m=m)
    keys = gen.keys(n, seed=42, dist=gen.DIST_SKEW, alpha=0.3, **gk)
    vals = gen.values(n, seed=42)
    ek, ev, eo = oracle.multisplit(keys, _to_oracle(bucket), vals)
    got_k = np.concatenate([np.load(tmp_path / f"k{r}.npy") for r in range(world)])
    assert [np.load(tmp_path / f"k{r}.npy").size for r in range(world)] == sizes  # output shard = input shard size
    assert np.array_equal(got_k, ek)
    if pairs:
        got_v = np.concatenate([np.load(tmp_path / f"v{r}.npy") for r in range(world)])
        assert np.array_equal(got_v, ev)
    for r in range(world):
        assert np.load(tmp_path / f"o{r}.npy").tolist() == eo.astype(np.uint64).tolist()


@pytest.mark.parametrize("G,m", [(1, 5), (2, 2), (4, 16), (8, 256), (5, 3)])
def test_shard_plan_consistency(G, m):
    rng = np.random.default_rng(G * 1000 + m)
    C = rng.integers(0, 50, (G, m)).astype(np.uint64)
    C[rng.integers(0, G)] = 0  # an empty shard
    n = C.sum(axis=1).astype(np.int64)
    plans = [sharded.shard_plan(C, r) for r in range(G)]
    for r in range(G):
        p = plans[r]
        # r's sends tile its local order contiguously, in destination order
        assert int(p["send_displs"][0]) == 0
        assert np.array_equal(np.cumsum(p["send_counts"].astype(np.int64))[:-1],
                              p["send_displs"][1:].astype(np.int64))
        assert int(p["send_counts"].sum()) == n[r]
        # what r receives from s is what s sends to r; r receives exactly its shard size
        for s in range(G):
            assert int(p["recv_counts"][s]) == int(plans[s]["send_counts"][r])
        assert int(p["recv_counts"].sum()) == n[r]
    # global bucket offsets = exclusive scan of the column sums (Eq.3 term 1)
    tot = C.sum(axis=0).astype(np.int64)
    assert plans[0]["global_offsets"].astype(np.int64).tolist() == np.concatenate([[0], np.cumsum(tot)]).tolist()
