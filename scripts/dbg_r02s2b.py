"""Same-process repeat of C3 identity m=256 pairs (uniform, skew, ...): mismatch details."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, paper_1701_01189_b200 as ms
from gen import device as gdev, inputs as gen
ms.device_init(0)
h = lambda t: t.cpu().numpy().view(np.uint32)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
m = 256
for it, dist in enumerate([0, 1, 0, 1, 1, 0]):
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(k, 0x5EED + m, dist=dist, alpha=0.1, kind=gen.IDENTITY, m=m)
    v = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.values_(v, 0x5EED + m, parity=True)
    kh, vh = h(k), h(v)
    ek, ev, eo = oracle.multisplit(kh, oracle.identity(m), vh)
    for rep in range(2):
        ko, vo, off = ms.multisplit(k, v, bucket=ms.Identity(m))
        torch.cuda.synchronize()
        a, b, o = h(ko), h(vo), h(off)
        res = dict(it=it, dist=dist, rep=rep, off_ok=bool(np.array_equal(o, eo)), kbad=int((a != ek).sum()), vbad=int((b != ev).sum()))
        if res["vbad"]:
            bad = np.nonzero(b != ev)[0]
            i = int(bad[0])
            bk = int(np.searchsorted(eo, i, side="right") - 1)
            res.update(first=i, last=int(bad[-1]), bucket=bk, pos_in_bucket=i - int(eo[bk]), got_src=int(b[i]), exp_src=int(ev[i]),
                       buckets_bad=np.unique(np.searchsorted(eo, bad, side="right") - 1)[:10].tolist())
            # got values are input indices: are they a permutation within the bucket?
            lo, hi = int(eo[bk]), int(eo[bk + 1])
            res["bucket_perm_ok"] = bool(np.array_equal(np.sort(b[lo:hi]), np.sort(ev[lo:hi])))
        print(json.dumps(res), flush=True)
        del ko, vo, off
