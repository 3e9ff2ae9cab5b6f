"""Sharded multisplit on one GPU with G virtual ranks: each rank's local
multisplit and receiver merge run as the real CUDA kernels; the all-gather and
all-to-all-v are done by slicing device tensors (the same split sizes the NCCL
path uses).  The concatenation of the output shards must equal the oracle's
stable multisplit of the concatenated input, element by element."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gen

pytestmark = pytest.mark.gpu
ms = pytest.importorskip("paper_1701_01189_b200")
from paper_1701_01189_b200 import sharded  # noqa: E402


def run_virtual(keys_np, vals_np, sizes, bucket):
    G = len(sizes)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    dev = torch.device("cuda")
    locals_ = []
    for r in range(G):
        k = torch.from_numpy(keys_np[bounds[r]:bounds[r + 1]].view(np.int32).copy()).to(dev)
        v = None if vals_np is None else torch.from_numpy(vals_np[bounds[r]:bounds[r + 1]].view(np.int32).copy()).to(dev)
        locals_.append(sharded._cuda_local(k, v, bucket))
    C = np.stack([(off[1:].to(torch.int64) - off[:-1].to(torch.int64)).cpu().numpy() for _, _, off in locals_])
    C = C.astype(np.uint64)
    plans = [sharded.shard_plan(C, r) for r in range(G)]
    outs_k, outs_v = [], []
    for r in range(G):
        # all-to-all-v: source s's range for r, packed in source order
        pk = [locals_[s][0][int(plans[s]["send_displs"][r]):int(plans[s]["send_displs"][r] + plans[s]["send_counts"][r])]
              for s in range(G)]
        rk = torch.cat(pk) if pk else torch.empty(0, dtype=torch.int32, device=dev)
        rv = None
        if vals_np is not None:
            pv = [locals_[s][1][int(plans[s]["send_displs"][r]):int(plans[s]["send_displs"][r] + plans[s]["send_counts"][r])]
                  for s in range(G)]
            rv = torch.cat(pv)
        ko, vo = sharded._cuda_merge(rk, rv, bucket, plans[r]["recv_displs"], plans[r]["merge_offsets"], G)
        outs_k.append(ko.cpu().numpy().view(np.uint32))
        if vo is not None:
            outs_v.append(vo.cpu().numpy().view(np.uint32))
    return outs_k, outs_v, plans[0]["global_offsets"]


@pytest.mark.parametrize("sizes", [[70000], [40000, 40000], [100003, 3, 50000], [30000] * 8,
                                   [0, 65536, 8193, 1, 77777]])
@pytest.mark.parametrize("m", [2, 33, 256])
def test_virtual_ranks(sizes, m):
    n = sum(sizes)
    ob = oracle.delta(m)
    keys = gen.keys(n, seed=n + m, kind=gen.DELTA, m=m, delta=ob.delta, dist=gen.DIST_SKEW, alpha=0.4)
    vals = gen.values(n, seed=1)
    ok, ov, goff = run_virtual(keys, vals, sizes, ms.Delta(m))
    ek, ev, eo = oracle.multisplit(keys, ob, vals)
    assert [x.size for x in ok] == sizes
    assert np.array_equal(np.concatenate(ok), ek) and np.array_equal(np.concatenate(ov), ev)
    assert goff.astype(np.int64).tolist() == eo.astype(np.int64).tolist()


def test_virtual_ranks_keys_identity():
    sizes = [50000, 12345, 99999]
    n = sum(sizes)
    keys = gen.keys(n, seed=5, kind=gen.IDENTITY, m=64)
    ok, _, _ = run_virtual(keys, None, sizes, ms.Identity(64))
    ek, _, _ = oracle.multisplit(keys, oracle.identity(64))
    assert np.array_equal(np.concatenate(ok), ek)
