"""Multisplit-SSSP on the bench R-MAT graph: time, iterations and work per (delta, K)."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1701_01189_b200 as ms
from gen.graphs import rmat_csr
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
V, rp, col, w = rmat_csr(scale, 5, 0x5EED, undirected=True)
cv = lambda a: torch.from_numpy(a.view(np.int32)).cuda()
R, C, W = cv(rp), cv(col), cv(w)
ms.device_init(0)
for delta, K in [(200, 10)]:
    ws = torch.empty(ms._lib.load().ms_sssp_workspace_size(V, col.size, K), dtype=torch.uint8, device="cuda")
    d, st = ms.sssp(R, C, W, 0, delta=delta, buckets=K, workspace=ws, stats=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ms.sssp(R, C, W, 0, delta=delta, buckets=K, out=d, workspace=ws); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    t = sorted(ts)[len(ts) // 2]
    print(json.dumps({"delta": delta, "K": K, "ms": round(t, 3), "MTEPS": round(col.size / t / 1e3, 1),
                      "us_per_iter": round(t * 1e3 / st["iterations"], 2), **st}), flush=True)
