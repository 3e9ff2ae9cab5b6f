"""Quick device-timed rates for a list of workload:m specs (no e2e, no CPU):
python scripts/quick_rates.py ms_pairs_os:256 sort_keys:256 ..."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from gen import device as gdev

dev = torch.device("cuda:0")
scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
flush = lambda: gdev.flush_(scratch)  # noqa: E731
hbm, _ = bench.load_peaks()
for spec in sys.argv[1:]:
    name, m = spec.split(":")
    m = int(m)
    wl = bench.WORKLOADS[name]
    run = bench.Runner(wl, m, dev)
    steps = 5 if wl["kind"] == "sort" else 10
    times, _, _ = bench.time_steps(run, steps, 3, flush, stage_events=False)
    t = sum(times) / len(times)
    rate = run.n / (t * 1e-3) / 1e9
    print(json.dumps({"case": spec, "rate": round(rate, 2), "unit": wl["unit"], "ms": round(t, 4),
                      "hbm_frac": round(rate * 1e9 * wl["bpe"] / (hbm * 1e9), 3)}), flush=True)
    del run
    torch.cuda.empty_cache()
