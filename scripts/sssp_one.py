import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1701_01189_b200 as ms
from gen.graphs import rmat_csr
V, rp, col, w = rmat_csr(20, 5, 0x5EED, undirected=True)
cv = lambda a: torch.from_numpy(a.view(np.int32)).cuda()
R, C, W = cv(rp), cv(col), cv(w)
ms.device_init(0)
d = ms.sssp(R, C, W, 0, delta=200, buckets=10)
torch.cuda.synchronize()
print("ok")
