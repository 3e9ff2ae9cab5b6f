import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1701_01189_b200 as ms
for m, n in ((257, 1), (257, 1000), (300, 1), (256, 1), (1000, 5)):
    r = np.random.default_rng(m)
    spl = np.sort(r.choice(1 << 32, size=m - 1, replace=False).astype(np.uint64)).astype(np.uint32)
    keys = torch.from_numpy(r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
    sp = torch.from_numpy(spl.view(np.int32)).cuda()
    try:
        ko, _, off = ms.multisplit(keys, None, bucket=ms.Splitters(sp))
        torch.cuda.synchronize()
        print("ok", m, n, flush=True)
    except Exception as e:
        print("FAIL", m, n, repr(e)[:300], flush=True)
        try:
            torch.cuda.synchronize()
        except Exception as e2:
            print("  sync:", repr(e2)[:200])
        break
