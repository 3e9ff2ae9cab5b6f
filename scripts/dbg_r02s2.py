"""Debug matrix for the wide (m > 32) pipeline: parity vs the oracle per case, in
one process per case (an illegal address kills the context)."""
import os, sys, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def one(n, m, pairs, kind, dist, rank_mode):
    import numpy as np, torch
    import oracle, paper_1701_01189_b200 as ms
    from gen import device as gdev, inputs as gen
    ms.device_init(0)
    if rank_mode:
        ms.set_option(0, 1)
    bits = m.bit_length() - 1
    if kind == "identity":
        ob, pb, gk = oracle.identity(m), ms.Identity(m), dict(kind=gen.IDENTITY, m=m)
    elif kind == "radix":
        ob, pb, gk = oracle.radix(0, bits), ms.Radix(0, bits), dict(kind=gen.RADIX, m=m, shift=0, bits=bits)
    else:
        ob = oracle.delta(m); pb = ms.Delta(m); gk = dict(kind=gen.DELTA, m=m, delta=ob.delta)
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(k, 0x5EED + m, dist=dist, alpha=0.1, **gk)
    v = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.values_(v, 0x5EED + m, parity=True)
    h = lambda t: t.cpu().numpy().view(np.uint32)
    kh, vh = h(k), h(v)
    ek, ev, eo = oracle.multisplit(kh, ob, vh if pairs else None)
    ko, vo, off = ms.multisplit(k, v if pairs else None, bucket=pb)
    torch.cuda.synchronize()
    a, o = h(ko), h(off)
    res = dict(offsets_ok=bool(np.array_equal(o, eo)), keys_bad=int((a != ek).sum()))
    if pairs:
        bv = h(vo) != ev
        res["vals_bad"] = int(bv.sum())
        if bv.any():
            i = int(np.nonzero(bv)[0][0])
            bk = int(np.searchsorted(eo, i, side="right") - 1)
            res["first_bad"] = i; res["bucket"] = bk; res["pos_in_bucket"] = i - int(eo[bk])
            res["tile_of_bad_val_src"] = int(h(vo)[i]) // 4096
            res["exp_src_tile"] = int(ev[i]) // 4096
    if res["keys_bad"]:
        i = int(np.nonzero(a != ek)[0][0]); res["first_bad_key"] = i
    if not res["offsets_ok"]:
        d = np.nonzero(o != eo)[0]; res["off_bad"] = d[:4].tolist()
    return res

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        n, m, pairs, kind, dist, rm = sys.argv[2:]
        print(json.dumps(one(int(n), int(m), pairs == "1", kind, int(dist), int(rm))))
        sys.exit(0)
    cases = []
    for n in (1 << 20, 1 << 24, 1 << 27):
        for m in (64, 256):
            for pairs in (0, 1):
                for kind in ("identity", "radix"):
                    for dist in (0, 1):
                        cases.append((n, m, pairs, kind, dist, 0))
    cases += [(1 << 27, 256, 1, "identity", 1, 1), (1 << 24, 256, 1, "identity", 1, 1),
              (1 << 25, 128, 0, "delta", 0, 0), (1 << 25, 128, 1, "delta", 0, 0),
              (1 << 25, 64, 1, "delta", 0, 0), (1 << 25, 256, 1, "delta", 0, 0)]
    for c in cases:
        r = subprocess.run([sys.executable, __file__, "one", *map(str, c)], capture_output=True, text=True, timeout=600)
        out = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip().splitlines()[-1][:200]
        print(c, out, flush=True)
