"""Sharded stable multisplit across the ranks of a torch.distributed group.

Eq.(3) of the paper with the GPUs as the first localization
level (L_0 = G ranks): rank s holds input shard s and receives output shard s
(the same global index range of the stable multisplit of the rank-order
concatenation of the shards).  Steps (include/multisplit.h, "Sharded
multisplit"):

  1. local stable multisplit of the shard on the GPU (ms_multisplit_*),
  2. all-gather of the G x m bucket counts (NCCL),
  3. ms_shard_plan on the host: all-to-all-v counts and the merge offsets,
  4. all-to-all-v of keys (and values) (NCCL): what rank s sends to rank d is
     one contiguous range of its local bucket order,
  5. receiver merge on the GPU (ms_shard_merge_*).

torch.distributed is the plumbing (process group, collectives); every step on
the data runs in libms kernels.  The ops of steps 1 and 5 are parameters only
so that the host logic can be exercised on CPU-only gloo groups in tests.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import check


def shard_plan(C: np.ndarray, rank: int) -> dict:
    """Host-side plan of rank `rank` from the gathered counts C (G x m): send/recv
    counts and displacements, merge offsets (G x m, uint32) and the global bucket
    offsets (m + 1)."""
    C = np.ascontiguousarray(C, dtype=np.uint64)
    G, m = C.shape
    sc = np.zeros(G, np.uint64)
    sd = np.zeros(G, np.uint64)
    rc = np.zeros(G, np.uint64)
    rd = np.zeros(G, np.uint64)
    mo = np.zeros((G, m), np.uint32)
    go = np.zeros(m + 1, np.uint64)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    check(_lib.load().ms_shard_plan(p(C), G, m, rank, p(sc), p(sd), p(rc), p(rd), p(mo), p(go)),
          "ms_shard_plan")
    return dict(send_counts=sc, send_displs=sd, recv_counts=rc, recv_displs=rd, merge_offsets=mo,
                global_offsets=go)


def _cuda_local(keys, values, bucket):
    from . import multisplit
    return multisplit(keys, values, bucket=bucket)


def _cuda_merge(keys_recv, vals_recv, bucket, recv_displs, merge_offsets, G):
    lib = _lib.load()
    n = keys_recv.numel()
    dev = keys_recv.device
    starts = torch.tensor(np.append(recv_displs, n).astype(np.int64), dtype=torch.int64)
    starts = starts.to(torch.int32).to(dev)
    offs = torch.from_numpy(merge_offsets.view(np.int32).copy()).to(dev)
    ko = torch.empty_like(keys_recv)
    vo = torch.empty_like(vals_recv) if vals_recv is not None else None
    fn = bucket.c()
    sp = torch.cuda.current_stream().cuda_stream
    if vals_recv is not None:
        check(lib.ms_shard_merge_pairs(keys_recv.data_ptr(), vals_recv.data_ptr(), n, ctypes.byref(fn),
                                       starts.data_ptr(), offs.data_ptr(), G, ko.data_ptr(), vo.data_ptr(),
                                       sp), "ms_shard_merge_pairs")
    else:
        check(lib.ms_shard_merge_keys(keys_recv.data_ptr(), n, ctypes.byref(fn), starts.data_ptr(),
                                      offs.data_ptr(), G, ko.data_ptr(), sp), "ms_shard_merge_keys")
    return ko, vo


def sharded_multisplit(keys: torch.Tensor, values: torch.Tensor | None, bucket, group=None, *,
                       local_op=None, merge_op=None):
    """Stable multisplit of the rank-order concatenation of every rank's shard.

    Returns (keys_out, values_out | None, global_bucket_offsets[m+1] as numpy uint64);
    keys_out is this rank's output shard (same length as its input shard)."""
    local_op = local_op or _cuda_local
    merge_op = merge_op or _cuda_merge
    G = dist.get_world_size(group)
    r = dist.get_rank(group)
    m = bucket.m
    # 1. local stable multisplit: local bucket order + the shard's bucket counts
    ko, vo, off = local_op(keys, values, bucket)
    counts = (off[1:].to(torch.int64) - off[:-1].to(torch.int64))
    # 2. all-gather of the counts (G x m)
    C = torch.empty(G * m, dtype=torch.int64, device=counts.device)
    dist.all_gather_into_tensor(C, counts.contiguous(), group=group)
    Ch = C.view(G, m).cpu().numpy().astype(np.uint64)
    # 3. plan (host)
    plan = shard_plan(Ch, r)
    send = [int(x) for x in plan["send_counts"]]
    recv = [int(x) for x in plan["recv_counts"]]
    # 4. all-to-all-v: rank r's local order is split into G consecutive ranges
    rk = torch.empty(sum(recv), dtype=keys.dtype, device=keys.device)
    dist.all_to_all_single(rk, ko, output_split_sizes=recv, input_split_sizes=send, group=group)
    rv = None
    if values is not None:
        rv = torch.empty(sum(recv), dtype=values.dtype, device=values.device)
        dist.all_to_all_single(rv, vo, output_split_sizes=recv, input_split_sizes=send, group=group)
    # 5. receiver merge
    out_k, out_v = merge_op(rk, rv, bucket, plan["recv_displs"], plan["merge_offsets"], G)
    return out_k, out_v, plan["global_offsets"]
