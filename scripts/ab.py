"""A/B timing of workloads under library options: python scripts/ab.py 'ms_keys:4,ms_keys:8' 'rank=0;rank=2'
Each case: parity of one call against the oracle, then the bench timing (L2 flushed, CUDA events)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench, oracle
import paper_1701_01189_b200 as ms
from gen import device as gdev

cases = [c.split(":") for c in sys.argv[1].split(",")]
variants = sys.argv[2].split(";") if len(sys.argv) > 2 else [""]
dev = torch.device("cuda", 0)
scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
flush = lambda: gdev.flush_(scratch)
hbm, _ = bench.load_peaks()
OPT = {"rank": 0, "runs": 1, "pipe": 2}
h = lambda t: t.cpu().numpy().view(np.uint32)
for name, m in cases:
    m = int(m)
    wl = bench.WORKLOADS[name]
    run = bench.Runner(wl, m, dev)
    for v in variants:
        for kv in filter(None, v.split("+")):
            k, x = kv.split("=")
            ms.set_option(OPT[k], int(x))
        ok = None
        if run.bucket is not None and 0 < wl["n"] <= (1 << 25):
            run.step(); torch.cuda.synchronize()
            ob = {"delta": lambda: oracle.delta(m), "identity": lambda: oracle.identity(m),
                  "radix": lambda: oracle.radix(0, m.bit_length() - 1),
                  "splitters": lambda: oracle.splitters(h(run.spl))}[wl["kind"]]()
            ek, ev, eo = oracle.multisplit(h(run.keys), ob, h(run.vals) if run.vals is not None else None)
            ok = bool(np.array_equal(h(run.ko), ek) and np.array_equal(h(run.off), eo) and
                      (run.vals is None or np.array_equal(h(run.vo), ev)))
        times, _, _ = bench.time_steps(run, 20, 3, flush, stage_events=False)
        _, st, _ = bench.time_steps(run, 5, 1, flush, stage_events=True)
        t = sum(times) / len(times)
        rate = run.n / (t * 1e-3) / (1e6 if wl["unit"] == "MTEPS" else 1e9)
        print(json.dumps({"case": f"{name}:{m}", "var": v or "default", "parity": ok, "rate": round(rate, 2),
                          "frac": round(rate * 1e9 * wl["bpe"] / (hbm * 1e9), 4),
                          "stage_ms": {k: round(x, 4) for k, x in (st or {}).items()}}), flush=True)
        for kv in filter(None, v.split("+")):
            k, _ = kv.split("=")
            ms.set_option(OPT[k], {"rank": 0, "runs": 1, "pipe": 0}[k])
    del run
    torch.cuda.empty_cache()
