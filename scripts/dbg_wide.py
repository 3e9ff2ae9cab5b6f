import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, paper_1701_01189_b200 as ms
from gen import inputs as gen
ms.device_init(0)
print("probe", ms._lib.load().ms_lane_ordered_increment())
def d(a): return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()
def h(t): return t.cpu().numpy().view(np.uint32)
for m in (64, 100, 128, 200, 255, 256):
    for n in (8192 * 3, 1 << 20):
        for pairs in (False, True):
            ob = oracle.delta(m)
            k = gen.keys(n, seed=1 + m, kind=gen.DELTA, m=m, delta=ob.delta)
            v = gen.values(n, seed=1)
            ek, ev, eo = oracle.multisplit(k, ob, v if pairs else None)
            ko, vo, off = ms.multisplit(d(k), d(v) if pairs else None, bucket=ms.Delta(m))
            a, o = h(ko), h(off)
            bad = np.nonzero(a != ek)[0]
            offok = np.array_equal(o, eo)
            msg = f"m={m} n={n} pairs={pairs} offsets_ok={offok} nbad={bad.size}"
            if bad.size:
                i = bad[0]
                bk = np.searchsorted(eo, i, side='right') - 1
                msg += f" first={i} bucket_of_pos={bk} got_bucket={ob and oracle.multisplit(a[i:i+1], ob)[2].argmax()}"
                if not offok:
                    db = np.nonzero(o != eo)[0]
                    msg += f" off_bad={db[:5]} got={o[db[:5]]} exp={eo[db[:5]]}"
            print(msg, flush=True)
