"""Sharded stable multisplit across the ranks of one node (one process per GPU).

Eq.(3) of the paper with the GPUs as the first localization
level (L_0 = G ranks): rank s holds input shard s and receives output shard s
(the same global index range of the stable multisplit of the rank-order
concatenation of the shards).  Every step runs inside libms
(include/multisplit.h, "Sharded multisplit as the library's own call"):
NCCL collectives and the fused peer-store scatter (KP) or the NCCL
send/receive path with the KX merge.  This module only creates the
communicator: rank 0's NCCL unique id is broadcast over a torch.distributed
process group (the plumbing), then every rank calls ms_comm_init.

    comm = sharded.Comm(group)                     # collective
    comm.register_output(out_keys, out_values)     # collective, once per buffer pair
    ko, vo, goff = sharded.multisplit(comm, keys, values, bucket=ms.Delta(256),
                                      out_keys=out_keys, out_values=out_values)

`exchange_reference` is the same exchange written with torch.distributed
collectives around the host plan (ms_shard_plan); the CPU tests run it on gloo
process groups with oracle stand-ins for the device steps, to check the plan
arithmetic across processes.  It is not used by the product path.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import check


class Comm:
    """An ms_comm over the ranks of `group` (collective).  `device` defaults to
    torch's current CUDA device."""

    def __init__(self, group=None, device: int | None = None):
        lib = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            check(lib.ms_comm_unique_id(uid), "ms_comm_unique_id")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        self._c = ctypes.c_void_p()
        check(lib.ms_comm_init(ctypes.byref(self._c), self.world, self.rank, uid, self.device), "ms_comm_init")
        self._windows = None

    def register_output(self, out_keys: torch.Tensor, out_values: torch.Tensor | None = None) -> None:
        """Make these output buffers the fused path's peer windows (collective)."""
        check(_lib.load().ms_comm_register_output(
            self._c, out_keys.data_ptr(), out_values.data_ptr() if out_values is not None else None,
            out_keys.numel()), "ms_comm_register_output")
        self._windows = (out_keys, out_values)  # keep them alive while registered

    def workspace_size(self, n_local: int, m: int, with_values: bool) -> int:
        return int(_lib.load().ms_sharded_workspace_size(self._c, n_local, m, int(with_values)))

    def check(self) -> None:
        """ms_comm_check: raise MultisplitError(MS_ERR_NCCL) if NCCL reported an async error."""
        check(_lib.load().ms_comm_check(self._c), "ms_comm_check")

    def abort(self) -> None:
        """ms_comm_abort: abort the NCCL communicator after a failure (then close())."""
        check(_lib.load().ms_comm_abort(self._c), "ms_comm_abort")

    def close(self) -> None:
        if self._c:
            check(_lib.load().ms_comm_destroy(self._c), "ms_comm_destroy")
            self._c = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass


def multisplit(comm: Comm, keys: torch.Tensor, values: torch.Tensor | None = None, *, bucket,
               out_keys: torch.Tensor | None = None, out_values: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None, stream=None):
    """ms_multisplit_{keys,pairs}_sharded: this rank's output shard (same length as its
    input shard) and the m+1 global bucket offsets (int64 tensor on the device)."""
    from . import _u32view, _workspace, _prepare, _stream_ptr
    lib = _lib.load()
    keys = _u32view(keys, "keys")
    dv = keys.device
    n = keys.numel()
    pairs = values is not None
    if pairs:
        values = _u32view(values, "values", dv, n)
    ko = _u32view(out_keys, "out_keys", dv, n) if out_keys is not None else torch.empty_like(keys)
    vo = None
    if pairs:
        vo = _u32view(out_values, "out_values", dv, n) if out_values is not None else torch.empty_like(values)
    goff = torch.empty(bucket.m + 1, dtype=torch.int64, device=dv)
    ws = _workspace(workspace, comm.workspace_size(n, bucket.m, pairs), dv)
    fn = bucket.c()
    _prepare(keys)
    with torch.cuda.device(dv):
        sp = _stream_ptr(stream, dv)
        if pairs:
            st = lib.ms_multisplit_pairs_sharded(comm._c, keys.data_ptr(), values.data_ptr(), ko.data_ptr(),
                                                 vo.data_ptr(), n, ctypes.byref(fn), goff.data_ptr(),
                                                 ws.data_ptr(), ws.numel(), sp)
        else:
            st = lib.ms_multisplit_keys_sharded(comm._c, keys.data_ptr(), ko.data_ptr(), n, ctypes.byref(fn),
                                                goff.data_ptr(), ws.data_ptr(), ws.numel(), sp)
    check(st, "ms_multisplit_pairs_sharded" if pairs else "ms_multisplit_keys_sharded")
    return ko, vo, goff


def shard_plan(C: np.ndarray, rank: int) -> dict:
    """Host-side plan of rank `rank` from the gathered counts C (G x m): send/recv
    counts and displacements, merge offsets (G x m, uint32) and the global bucket
    offsets (m + 1) -- ms_shard_plan, the plan the library's NCCL path uses."""
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


def exchange_reference(keys: torch.Tensor, values: torch.Tensor | None, bucket, local_op, merge_op,
                       group=None):
    """The NCCL path's exchange written with torch.distributed collectives (test model).

    local_op(keys, values, bucket) -> (local order keys, values, m+1 offsets);
    merge_op(keys_recv, vals_recv, bucket, recv_displs, merge_offsets, G) -> (keys, values).
    Returns (keys_out, values_out | None, global bucket offsets as numpy uint64)."""
    G = dist.get_world_size(group)
    r = dist.get_rank(group)
    m = bucket.m
    ko, vo, off = local_op(keys, values, bucket)
    counts = off[1:].to(torch.int64) - off[:-1].to(torch.int64)
    C = torch.empty(G * m, dtype=torch.int64, device=counts.device)
    dist.all_gather_into_tensor(C, counts.contiguous(), group=group)
    plan = shard_plan(C.view(G, m).cpu().numpy().astype(np.uint64), r)
    send = [int(x) for x in plan["send_counts"]]
    recv = [int(x) for x in plan["recv_counts"]]
    rk = torch.empty(sum(recv), dtype=keys.dtype, device=keys.device)
    dist.all_to_all_single(rk, ko, output_split_sizes=recv, input_split_sizes=send, group=group)
    rv = None
    if values is not None:
        rv = torch.empty(sum(recv), dtype=values.dtype, device=values.device)
        dist.all_to_all_single(rv, vo, output_split_sizes=recv, input_split_sizes=send, group=group)
    out_k, out_v = merge_op(rk, rv, bucket, plan["recv_displs"], plan["merge_offsets"], G)
    return out_k, out_v, plan["global_offsets"]


def virtual_ranks(keys: list[torch.Tensor], values: list[torch.Tensor] | None, bucket,
                  outs_k: list[torch.Tensor] | None = None, outs_v: list[torch.Tensor] | None = None):
    """The fused path KP for G virtual ranks on one GPU (ms_shard_prescan /
    ms_shard_scatter; the all-gather becomes the shared count matrix C).  Returns
    (output shards of keys, of values or None, global bucket offsets int64)."""
    from . import _u32view, _stream_ptr, _prepare
    lib = _lib.load()
    G = len(keys)
    dv = keys[0].device
    m = bucket.m
    pairs = values is not None
    fn = bucket.c()
    outs_k = outs_k or [torch.empty_like(k) for k in keys]
    outs_v = (outs_v or [torch.empty_like(v) for v in values]) if pairs else None
    C = torch.zeros(G * m, dtype=torch.int32, device=dv)
    goff = torch.empty(m + 1, dtype=torch.int64, device=dv)
    _prepare(keys[0])
    sp = _stream_ptr(None, dv)
    wss = []
    for r in range(G):
        k = _u32view(keys[r], "keys", dv)
        ws = torch.empty(max(1, int(lib.ms_shard_workspace_size(k.numel(), m, G, int(pairs)))),
                         dtype=torch.uint8, device=dv)
        wss.append(ws)
        check(lib.ms_shard_prescan(k.data_ptr(), k.numel(), ctypes.byref(fn), int(pairs), G,
                                   C.data_ptr() + 4 * r * m, ws.data_ptr(), ws.numel(), sp), "ms_shard_prescan")
    pk = (ctypes.c_void_p * G)(*[o.data_ptr() for o in outs_k])
    pv = (ctypes.c_void_p * G)(*[o.data_ptr() for o in outs_v]) if pairs else None
    for r in range(G):
        check(lib.ms_shard_scatter(keys[r].data_ptr(), values[r].data_ptr() if pairs else None, keys[r].numel(),
                                   ctypes.byref(fn), C.data_ptr(), G, r, pk, pv,
                                   goff.data_ptr() if r == 0 else None, wss[r].data_ptr(), wss[r].numel(), sp),
              "ms_shard_scatter")
    return outs_k, outs_v, goff
