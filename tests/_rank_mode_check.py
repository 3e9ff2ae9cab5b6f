"""Subprocess body of test_gpu_rank_modes.py: one kf_meta rank mode (selected by
MS_META_RANK / MS_META_PROD in the environment, read once per process) against
the oracle on multi-tile inputs that span ragged tails, several m <= 32 and
skewed bucket distributions.  Exit code 0 = every case bit-exact."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1701_01189_b200 as ms  # noqa: E402
from gen import inputs as gen  # noqa: E402


def main():
    bad = 0
    for m in (3, 5, 8, 13, 16, 17, 32):
        for n, pairs, dist in ((3 * 8192 + 77, False, gen.DIST_UNIFORM), (5 * 4096 + 1, True, gen.DIST_UNIFORM),
                               (40000, False, gen.DIST_SKEW), (9000, True, gen.DIST_BINOMIAL)):
            ob = oracle.delta(m)
            k = gen.keys(n, seed=m * 7 + n, kind=gen.DELTA, m=m, delta=ob.delta, dist=dist, alpha=0.1)
            v = gen.values(n, seed=3) if pairs else None
            ek, ev, eo = oracle.multisplit(k, ob, v)
            kd = torch.from_numpy(k.view(np.int32)).cuda()
            vd = torch.from_numpy(v.view(np.int32)).cuda() if pairs else None
            ko, vo, off = ms.multisplit(kd, vd, bucket=ms.Delta(m))
            ok = np.array_equal(ko.cpu().numpy().view(np.uint32), ek) and \
                np.array_equal(off.cpu().numpy().view(np.uint32), eo) and \
                (not pairs or np.array_equal(vo.cpu().numpy().view(np.uint32), ev))
            if not ok:
                bad += 1
                print("MISMATCH", os.environ.get("MS_META_RANK"), m, n, pairs, dist)
    print("ok" if bad == 0 else f"{bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
