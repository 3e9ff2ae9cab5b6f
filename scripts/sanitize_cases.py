"""Small invocations of every libms kernel for compute-sanitizer (memcheck,
racecheck, synccheck): KM + kf_meta (m <= 32; ballot / increment / peer-mask
ranks, producer-warp and per-element stores), KU + KR + kf_fused (m > 32 and
the single-CTA path), KH + KG + kf_fused (the tile pipeline and the stage API),
the radix sort, KX (shard merge), kh_histogram, splitter buckets, the m > 256 path
(KB / KO / KGA), Multisplit-SSSP; n in {1, 1000, 2^16 (+ ragged)}.
Each result is compared with the oracle (exit code 1 on a mismatch)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1701_01189_b200 as ms  # noqa: E402
from paper_1701_01189_b200 import sharded  # noqa: E402
from gen import inputs as gen  # noqa: E402

lib = ms._lib
bad = 0


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def h(t):
    return t.cpu().numpy().view(np.uint32)


def check(name, ok):
    global bad
    if not ok:
        bad += 1
        print("MISMATCH", name, flush=True)


ms.device_init(0)
NS = [1, 1000, (1 << 16) + 77]
for rank in (lib.MS_RANK_AUTO, lib.MS_RANK_PEER_MASKS):
    ms.set_option(lib.MS_OPT_RANK, rank)
    for stores in (1, 0):
        ms.set_option(lib.MS_OPT_RUN_STORES, stores)
        for m in (2, 8, 32, 64, 256):
            for n in NS:
                for pairs in (False, True):
                    ob = oracle.delta(m)
                    k = gen.keys(n, seed=m + n, kind=gen.DELTA, m=m, delta=ob.delta, dist=gen.DIST_SKEW, alpha=0.3)
                    v = gen.values(n, seed=1) if pairs else None
                    ek, ev, eo = oracle.multisplit(k, ob, v)
                    ko, vo, off = ms.multisplit(d(k), d(v) if pairs else None, bucket=ms.Delta(m))
                    check(f"ms r{rank} s{stores} m{m} n{n} p{pairs}",
                          np.array_equal(h(ko), ek) and np.array_equal(h(off), eo) and
                          (not pairs or np.array_equal(h(vo), ev)))
ms.set_option(lib.MS_OPT_RANK, lib.MS_RANK_AUTO)
ms.set_option(lib.MS_OPT_RUN_STORES, 1)
# unaligned inputs (no TMA loads) and outputs
for m in (4, 16, 100):
    n = 5 * 8192 + 3
    ob = oracle.delta(m)
    k = gen.keys(n + 1, seed=m, kind=gen.DELTA, m=m, delta=ob.delta)
    v = gen.values(n + 1, seed=2)
    ek, ev, _ = oracle.multisplit(k[1:], ob, v[1:])
    ko, vo, _ = ms.multisplit(d(k)[1:], d(v)[1:], bucket=ms.Delta(m))
    check(f"unaligned m{m}", np.array_equal(h(ko), ek) and np.array_equal(h(vo), ev))
# the paper's tile pipeline (KH -> KG -> kf_fused) and the stage API
ms.set_option(lib.MS_OPT_PIPELINE, lib.MS_PIPELINE_TILE)
for m in (2, 37, 256):
    n = 9 * 8192 + 5
    ob = oracle.delta(m)
    k = gen.keys(n, seed=m, kind=gen.DELTA, m=m, delta=ob.delta)
    ek, _, eo = oracle.multisplit(k, ob)
    ko, _, off = ms.multisplit(d(k), None, bucket=ms.Delta(m))
    check(f"tile pipeline m{m}", np.array_equal(h(ko), ek) and np.array_equal(h(off), eo))
ms.set_option(lib.MS_OPT_PIPELINE, lib.MS_PIPELINE_LEVEL0)
for m in (3, 256):
    k = gen.keys(50000, seed=3)
    H = ms.prescan(d(k), ms.Delta(m), tile=1000)
    G, off = ms.scan(H)
    Hn = oracle.tile_histogram(k, oracle.delta(m), 1000)
    check(f"stage m{m}", np.array_equal(h(H).reshape(Hn.shape), Hn))
# radix sort (8-bit and default digits), identity key-domain flag
for r in (8, 5):
    for n in NS:
        k = gen.keys(n, seed=r + n)
        v = gen.values(n, seed=1)
        ek, ev = oracle.radix_sort(k, v)
        ko, vo = ms.radix_sort(d(k), d(v), bits_per_pass=r)
        check(f"sort r{r} n{n}", np.array_equal(h(ko), ek) and np.array_equal(h(vo), ev))
k = gen.keys(3000, seed=1, kind=gen.IDENTITY, m=10)
k[77] = 10
ms.multisplit(d(k), None, bucket=ms.Identity(10))
check("domain flag", ms.device_status() == lib.MS_ERR_KEY_DOMAIN)
# sharded: the fused KP path (ms_shard_prescan / ms_shard_scatter) with 3 virtual
# ranks, and the NCCL path's plan + KX merge (ms_shard_merge_keys)
import ctypes  # noqa: E402
for G, m in ((3, 16), (3, 64)):
    ob = oracle.delta(m)
    shards = [gen.keys(20000 + 7 * r, seed=r, kind=gen.DELTA, m=m, delta=ob.delta) for r in range(G)]
    vals = [gen.values(s.size, seed=r) for r, s in enumerate(shards)]
    ok, ov, _ = sharded.virtual_ranks([d(s) for s in shards], [d(v) for v in vals], ms.Delta(m))
    ek, ev, _ = oracle.multisplit(np.concatenate(shards), ob, np.concatenate(vals))
    check(f"kp m{m}", np.array_equal(np.concatenate([h(x) for x in ok]), ek) and
          np.array_equal(np.concatenate([h(x) for x in ov]), ev))
    loc = [ms.multisplit(d(s), None, bucket=ms.Delta(m)) for s in shards]
    C = np.stack([np.diff(h(o).astype(np.int64)) for _, _, o in loc]).astype(np.uint64)
    out = []
    for r in range(G):
        plan = sharded.shard_plan(C, r)
        parts = []
        for q in range(G):
            sp = sharded.shard_plan(C, q)
            lo, cnt = int(sp["send_displs"][r]), int(sp["send_counts"][r])
            parts.append(loc[q][0][lo:lo + cnt])
        rk = torch.cat(parts)
        starts = d(np.append(plan["recv_displs"], rk.numel()).astype(np.uint32))
        offs = d(plan["merge_offsets"])
        ko = torch.empty_like(rk)
        fn = ms.Delta(m).c()
        lib.check(lib.load().ms_shard_merge_keys(rk.data_ptr(), rk.numel(), ctypes.byref(fn), starts.data_ptr(),
                                                 offs.data_ptr(), G, ko.data_ptr(), None))
        out.append(h(ko))
    check(f"shard merge m{m}", np.array_equal(np.concatenate(out), ek))
# histogram
x = gen.floats(70001, 5)
spl = gen.splitters(37, 5)
check("hist even", np.array_equal(h(ms.histogram_even(d(x.view(np.uint32)).view(torch.float32), 37, 0.0, 1024.0)),
                                  oracle.histogram_even(x, 37, 0.0, 1024.0)))
check("hist range", np.array_equal(h(ms.histogram_range(d(x.view(np.uint32)).view(torch.float32),
                                                        d(spl.view(np.uint32)).view(torch.float32))),
                                   oracle.histogram_range(x, spl)))
# splitter buckets (every kernel stages the table), m > 256 (bucket-id pass, two radix
# passes, offsets, gather), Multisplit-SSSP (splitters + relax)
for m in (8, 37, 256):
    spl = np.sort(np.random.default_rng(m).choice(1 << 32, m - 1, replace=False).astype(np.uint64)).astype(np.uint32)
    for n in (1000, (1 << 16) + 77):
        k = gen.keys(n, seed=m + 5)
        v = gen.values(n, seed=3)
        ek, ev, eo = oracle.multisplit(k, oracle.splitters(spl), v)
        ko, vo, off = ms.multisplit(d(k), d(v), bucket=ms.Splitters(d(spl)))
        check(f"splitters m{m} n{n}", np.array_equal(h(ko), ek) and np.array_equal(h(vo), ev) and
              np.array_equal(h(off), eo))
for ob, pb in ((oracle.delta(1000), ms.Delta(1000)), (oracle.radix(2, 12), ms.Radix(2, 12))):
    n = 30011
    k = gen.keys(n, seed=11)
    v = gen.values(n, seed=4)
    ek, ev, eo = oracle.multisplit(k, ob, v)
    ko, vo, off = ms.multisplit(d(k), d(v), bucket=pb)
    check(f"large m{ob.m}", np.array_equal(h(ko), ek) and np.array_equal(h(vo), ev) and np.array_equal(h(off), eo))
from gen.graphs import rmat_csr  # noqa: E402
V, rp, col, w = rmat_csr(9, 8, seed=2)
dist = ms.sssp(d(rp), d(col), d(w), 0, delta=50)
check("sssp", np.array_equal(h(dist), oracle.sssp(rp, col, w, 0)))
torch.cuda.synchronize()
print("sanitize cases:", "ok" if bad == 0 else f"{bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
