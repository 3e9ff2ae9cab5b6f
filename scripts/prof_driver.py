"""Minimal driver for ncu: runs one workload a few times (no timing, no sweep)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="ms_keys")
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
wl = bench.WORKLOADS[a.workload]
run = bench.Runner(wl, a.m or wl["m"], torch.device("cuda"))
for _ in range(a.reps):
    run.step()
torch.cuda.synchronize()
print("ok", a.workload, a.m)
