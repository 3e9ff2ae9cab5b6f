#!/usr/bin/env python3
"""bench.py -- throughput of the B200 stable multisplit (arXiv 1701.01189).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload NAME] [--m M] [--no-sweep]

A step is one full multisplit (prescan -> scan -> postscan, SURVEY.md §8(a)
rows a1-a5) of one synthetic batch resident in HBM; the radix-sort workloads'
step is one 4-pass sort (row a6).  The default workload is BASELINE.json
configs[1], key-only multisplit of n = 2^25 uniform uint32 keys into m = 32
delta buckets (the north_star gate "key-only multisplit at m <= 32").  L2 is
flushed (512 MiB write, untimed) before every timed step; each step is timed
with CUDA events on the launching stream.  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, plain single-threaded C) on
a bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
NOMINAL_HBM_GBS = 8000.0   # nominal B200 HBM3e (context: SURVEY 8(d) asks for both fractions)


def kernel_name(m: int) -> str:
    """The postscan kernel (dominant kernel) of the pipeline libms picks for m."""
    if m <= 32:
        return "kf_meta (KF: rank + in-place reorder + coalesced / run stores; prescan KM)"
    return "kf_meta_wide (KF: packed-increment rank + in-place reorder + coalesced stores; prescan KMW, scan KR)"

# workload -> (n, pairs, kind, default m, metric unit, algorithmic bytes per element)
# Algorithmic bytes: the paper's speed-of-light accounting: keys are
# read twice and written once (12 B), pairs 20 B; sort = 4 passes of that.
WORKLOADS = {
    "ms_keys": dict(n=1 << 25, pairs=False, kind="delta", m=32, unit="Gkeys/s", bpe=12,
                    desc="key-only multisplit, n=2^25 uniform uint32, delta buckets (configs[1])"),
    "ms_pairs": dict(n=1 << 25, pairs=True, kind="delta", m=32, unit="Gpairs/s", bpe=20,
                     desc="key-value multisplit, n=2^25 uniform uint32, delta buckets (configs[1])"),
    "ms_pairs_c3": dict(n=1 << 27, pairs=True, kind="identity", m=256, unit="Gpairs/s", bpe=20,
                        desc="key-value multisplit, n=2^27, identity buckets (configs[2])"),
    "ms_pairs_c3_skew": dict(n=1 << 27, pairs=True, kind="identity", m=256, unit="Gpairs/s", bpe=20,
                             dist="skew", desc="key-value multisplit, n=2^27, identity, 90% one bucket (configs[2])"),
    "ms_pairs_c3_radix": dict(n=1 << 27, pairs=True, kind="radix", m=256, unit="Gpairs/s", bpe=20,
                              desc="key-value multisplit, n=2^27, radix-digit buckets (low bits) (configs[2])"),
    "ms_pairs_c3_radix_skew": dict(n=1 << 27, pairs=True, kind="radix", m=256, unit="Gpairs/s", bpe=20,
                                   dist="skew", desc="key-value multisplit, n=2^27, radix digits, 90% one bucket"),
    "ms_keys_c1": dict(n=1 << 10, pairs=False, kind="delta", m=2, unit="Gkeys/s", bpe=12,
                       desc="key-only multisplit, n=2^10 uniform uint32, m=2 delta buckets (configs[0])"),
    "ms_sharded_c5": dict(n=1 << 30, pairs=True, kind="delta", m=256, unit="Gpairs/s", bpe=20,
                          desc="sharded key-value multisplit, n=2^30 pairs in total over the ranks, m=256 "
                               "delta buckets (configs[4]); n is per job, split evenly", strong=True),
    # the sorts' default path is the one-pass pipeline (f1): every digit histogram in
    # one read, then one fused look-back pass per digit (bpe_f1 = 36 / 68 B); bpe
    # stays the paper-faithful accounting (each pass a full multisplit, 48 / 80 B)
    "sort_keys": dict(n=1 << 28, pairs=False, kind="sort", m=256, unit="Gkeys/s", bpe=48, bpe_f1=36,
                      desc="multisplit LSD radix sort, 2^28 uint32 keys, 4 x 8-bit (configs[3])"),
    "sort_pairs": dict(n=1 << 28, pairs=True, kind="sort", m=256, unit="Gpairs/s", bpe=80, bpe_f1=68,
                       desc="multisplit LSD radix sort, 2^28 pairs, 4 x 8-bit (configs[3])"),
    "sort_keys_passes": dict(n=1 << 28, pairs=False, kind="sort", m=256, unit="Gkeys/s", bpe=48,
                             opts={"MS_OPT_SORT": "MS_SORT_PASSES"},
                             desc="multisplit LSD radix sort, 2^28 keys, 4 x 8-bit, each pass a full multisplit"),
    "sort_pairs_passes": dict(n=1 << 28, pairs=True, kind="sort", m=256, unit="Gpairs/s", bpe=80,
                              opts={"MS_OPT_SORT": "MS_SORT_PASSES"},
                              desc="multisplit LSD radix sort, 2^28 pairs, 4 x 8-bit, each pass a full multisplit"),
    # the one-pass multisplit (f1, MS_PIPELINE_ONESWEEP): bucket counts + one fused kernel
    "ms_keys_os": dict(n=1 << 25, pairs=False, kind="delta", m=32, unit="Gkeys/s", bpe=12,
                       opts={"MS_OPT_PIPELINE": "MS_PIPELINE_ONESWEEP"},
                       desc="key-only multisplit, n=2^25, delta buckets, one-pass pipeline (f1)"),
    "ms_pairs_os": dict(n=1 << 25, pairs=True, kind="delta", m=32, unit="Gpairs/s", bpe=20,
                        opts={"MS_OPT_PIPELINE": "MS_PIPELINE_ONESWEEP"},
                        desc="key-value multisplit, n=2^25, delta buckets, one-pass pipeline (f1)"),
    "ms_pairs_c3_os": dict(n=1 << 27, pairs=True, kind="identity", m=256, unit="Gpairs/s", bpe=20,
                           opts={"MS_OPT_PIPELINE": "MS_PIPELINE_ONESWEEP"},
                           desc="key-value multisplit, n=2^27, identity buckets, one-pass pipeline (f1)"),
    "ms_pairs_c3_skew_os": dict(n=1 << 27, pairs=True, kind="identity", m=256, unit="Gpairs/s", bpe=20,
                                dist="skew", opts={"MS_OPT_PIPELINE": "MS_PIPELINE_ONESWEEP"},
                                desc="key-value multisplit, n=2^27, identity, 90% one bucket, one-pass (f1)"),
    "ms_pairs_level0": dict(n=1 << 25, pairs=True, kind="delta", m=32, unit="Gpairs/s", bpe=20,
                            opts={"MS_OPT_PIPELINE": "MS_PIPELINE_LEVEL0"},
                            desc="key-value multisplit, n=2^25, delta buckets, two-kernel level-0 pipeline"),
    # the same sorts with 5-bit digits: 7 passes through the m <= 32 pipeline
    # (the paper's Table 8 sweeps r); bpe counts the 7 passes
    "sort_keys_r5": dict(n=1 << 28, pairs=False, kind="sort", m=32, bits=5, unit="Gkeys/s", bpe=84,
                         desc="multisplit LSD radix sort, 2^28 uint32 keys, 6 x 5-bit + 1 x 2-bit"),
    "sort_pairs_r5": dict(n=1 << 28, pairs=True, kind="sort", m=32, bits=5, unit="Gpairs/s", bpe=140,
                          desc="multisplit LSD radix sort, 2^28 pairs, 6 x 5-bit + 1 x 2-bit"),
    # device-wide histogram (Sec.7.3): 2^25 binary32 samples U[0,1024)
    "hist_even": dict(n=1 << 25, pairs=False, kind="hist_even", m=256, unit="Gsamples/s", bpe=4,
                      desc="device-wide Even histogram, 2^25 floats U[0,1024) (Sec.7.3, f2)"),
    "hist_range": dict(n=1 << 25, pairs=False, kind="hist_range", m=256, unit="Gsamples/s", bpe=4,
                       desc="device-wide Range histogram, 2^25 floats U[0,1024), m-1 random splitters (f2)"),
    # Multisplit-SSSP (Sec.7.2, f4): R-MAT scale 20 (1 M vertices), 5 edges per vertex made
    # undirected (10.5 M arcs, average degree 10; the paper's rmat: 0.8 M vertices, average
    # degree 12); weights 0..1000; source 0; delta 200 (measured best of 50..1000), 10 buckets
    "sssp_rmat": dict(n=0, pairs=False, kind="sssp", m=10, unit="MTEPS", bpe=0, scale=20, ef=5,
                      delta=200, desc="Multisplit-SSSP on an undirected R-MAT graph, scale 20, "
                                      "edge factor 5, weights 0..1000 (Sec.7.2, f4)"),
    # splitter buckets (f3): m-1 random sorted splitters over uniform keys
    "ms_keys_spl": dict(n=1 << 25, pairs=False, kind="splitters", m=32, unit="Gkeys/s", bpe=12,
                        desc="key-only multisplit, n=2^25 uniform uint32, m-1 random splitters (f3)"),
    "ms_pairs_spl": dict(n=1 << 25, pairs=True, kind="splitters", m=256, unit="Gpairs/s", bpe=20,
                         desc="key-value multisplit, n=2^25 uniform uint32, m-1 random splitters (f3)"),
    # m > 256 (f3, Sec.6.3): delta buckets, LSD over the bucket id's 8-bit digits
    "ms_keys_large": dict(n=1 << 25, pairs=False, kind="delta", m=4096, unit="Gkeys/s", bpe=12,
                          desc="key-only multisplit, n=2^25 uniform uint32, m > 256 delta buckets (f3)"),
    "ms_pairs_large": dict(n=1 << 25, pairs=True, kind="delta", m=4096, unit="Gpairs/s", bpe=20,
                           desc="key-value multisplit, n=2^25 uniform uint32, m > 256 delta buckets (f3)"),
    "sort_keys_r4": dict(n=1 << 28, pairs=False, kind="sort", m=16, bits=4, unit="Gkeys/s", bpe=96,
                         desc="multisplit LSD radix sort, 2^28 uint32 keys, 8 x 4-bit"),
    "sort_pairs_r4": dict(n=1 << 28, pairs=True, kind="sort", m=16, bits=4, unit="Gpairs/s", bpe=160,
                          desc="multisplit LSD radix sort, 2^28 pairs, 8 x 4-bit"),
}
SEED = 0x5EED


def metric_name(wl, name, m):
    k = wl["kind"]
    if k == "sort":
        return f"radix sort {wl['unit']} ({name})"
    if k == "sssp":
        return f"Multisplit-SSSP {wl['unit']} ({name}, K={m} buckets)"
    if k.startswith("hist"):
        return f"histogram {wl['unit']} ({name}, m={m})"
    return f"multisplit {wl['unit']} ({name}, m={m})"


def load_peaks():
    if os.path.exists(PEAKS_PATH):
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy test)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def load_traffic(key):
    if os.path.exists(TRAFFIC_PATH):
        with open(TRAFFIC_PATH) as f:
            return json.load(f).get(key)
    return None


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML in a thread during the timed region."""

    def __init__(self, index: int, period_s: float = 0.001):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self.index = period_s, index
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)

    _REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
                0x2: "applications_clocks_setting", 0x100: "sync_boost", 0x10: "display_clock_setting"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self._ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self._ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- our arm
class Runner:
    """Holds device inputs/outputs for one workload and runs one step per call."""

    def __init__(self, wl: dict, m: int, dev, rank: int = 0, world: int = 1):
        import torch
        import paper_1701_01189_b200 as ms
        from gen import device as gdev
        from gen import inputs as gen

        self.torch, self.ms, self.wl, self.m = torch, ms, wl, m
        self.world = world
        # N > 1: the sharded multisplit (all-gather of counts + all-to-all-v over
        # NCCL); weak scaling (n per rank) unless the workload fixes the job size
        n = wl["n"] // world if wl.get("strong") else wl["n"]
        self.n = n
        kind = wl["kind"]
        dist = {"skew": gen.DIST_SKEW, "binomial": gen.DIST_BINOMIAL}.get(wl.get("dist"), gen.DIST_UNIFORM)
        self.keys = torch.empty(n, dtype=torch.int32, device=dev)
        if kind == "delta":
            self.bucket = ms.Delta(m)
            gdev.keys_(self.keys, SEED + rank, kind=gen.DELTA, m=m, delta=self.bucket.delta, dist=dist, alpha=0.1)
        elif kind == "identity":
            self.bucket = ms.Identity(m)
            gdev.keys_(self.keys, SEED + rank, kind=gen.IDENTITY, m=m, dist=dist, alpha=0.1)
        elif kind == "radix":
            bits = m.bit_length() - 1
            self.bucket = ms.Radix(0, bits)
            gdev.keys_(self.keys, SEED + rank, kind=gen.RADIX, m=m, shift=0, bits=bits, dist=dist, alpha=0.1)
        elif kind == "splitters":
            import numpy as np
            r = np.random.default_rng(SEED + m)
            spl = np.sort(r.choice(1 << 32, size=m - 1, replace=False).astype(np.uint64)).astype(np.uint32)
            self.spl = torch.from_numpy(spl.view(np.int32)).to(dev)
            self.bucket = ms.Splitters(self.spl)
            gdev.keys_(self.keys, SEED + rank)
        elif kind == "sssp":
            from gen.graphs import rmat_csr
            import numpy as np
            self.bucket = None
            V, rp, col, w = rmat_csr(wl["scale"], wl["ef"], SEED, undirected=True)
            self.graph_host = (rp, col, w)
            cv = lambda a: torch.from_numpy(a.view(np.int32)).to(dev)  # noqa: E731
            self.rp, self.col, self.w = cv(rp), cv(col), cv(w)
            self.dist = torch.empty(V, dtype=torch.int32, device=dev)
            n = self.n = int(col.size)  # arcs: the MTEPS numerator
        elif kind.startswith("hist"):
            import numpy as np
            self.bucket = None
            self.samples = torch.from_numpy(gen.floats(n, SEED + rank)).to(dev)
            self.splitters = torch.from_numpy(gen.splitters(m, SEED)).to(dev)
            self.counts = torch.empty(m, dtype=torch.int32, device=dev)
        else:  # sort
            self.bucket = None
            gdev.keys_(self.keys, SEED + rank)
        self.vals = None
        if wl["pairs"]:
            self.vals = torch.empty(n, dtype=torch.int32, device=dev)
            gdev.values_(self.vals, SEED + rank, parity=False)
        self.ko = torch.empty_like(self.keys)
        self.vo = torch.empty_like(self.vals) if self.vals is not None else None
        self.off = torch.empty(m + 1, dtype=torch.int32, device=dev)
        if kind == "sssp":
            self.ws = torch.empty(ms._lib.load().ms_sssp_workspace_size(self.rp.numel() - 1, n, m),
                                  dtype=torch.uint8, device=dev)
        elif kind == "sort":
            self.ws = torch.empty(ms.radix_sort_workspace_size(n, wl["pairs"]), dtype=torch.uint8, device=dev)
        elif world > 1:
            from paper_1701_01189_b200 import sharded
            self.comm = sharded.Comm()
            self.comm.register_output(self.ko, self.vo)
            self.ws = torch.empty(max(1, self.comm.workspace_size(n, m, wl["pairs"])), dtype=torch.uint8,
                                  device=dev)
        else:
            self.ws = torch.empty(max(1, ms.workspace_size(n, m, wl["pairs"])), dtype=torch.uint8, device=dev)
        ms.device_init(dev.index)

    def sssp_stats(self):
        _, st = self.ms.sssp(self.rp, self.col, self.w, 0, delta=self.wl["delta"], buckets=self.m,
                             out=self.dist, workspace=self.ws, stats=True)
        return st

    def step(self, keys=None, ko=None):
        opts = self.wl.get("opts")
        if not opts:
            return self._step(keys, ko)
        lib = self.ms._lib
        saved = {o: self.ms.get_option(getattr(lib, o)) for o in opts}
        for o, v in opts.items():
            self.ms.set_option(getattr(lib, o), getattr(lib, v))
        try:
            return self._step(keys, ko)
        finally:
            for o, v in saved.items():
                self.ms.set_option(getattr(lib, o), v)

    def _step(self, keys=None, ko=None):
        keys = self.keys if keys is None else keys
        ko = self.ko if ko is None else ko
        if self.world > 1:  # the library's sharded call (fused KP path: registered windows)
            from paper_1701_01189_b200 import sharded
            sharded.multisplit(self.comm, keys, self.vals, bucket=self.bucket, out_keys=ko,
                               out_values=self.vo, workspace=self.ws)
            return
        if self.wl["kind"] == "sssp":
            self.ms.sssp(self.rp, self.col, self.w, 0, delta=self.wl["delta"], buckets=self.m,
                         out=self.dist, workspace=self.ws)
            return
        if self.wl["kind"] == "hist_even":
            self.ms.histogram_even(self.samples, self.m, 0.0, 1024.0, out=self.counts)
        elif self.wl["kind"] == "hist_range":
            self.ms.histogram_range(self.samples, self.splitters, out=self.counts)
        elif self.bucket is None:
            self.ms.radix_sort(keys, self.vals, bits_per_pass=self.wl.get("bits", 8), out_keys=ko,
                               out_values=self.vo, workspace=self.ws)
        else:
            self.ms.multisplit(keys, self.vals, bucket=self.bucket, out_keys=ko, out_values=self.vo,
                               out_offsets=self.off, workspace=self.ws)


def time_steps(run: Runner, steps: int, warmup: int, flush, stage_events: bool = True):
    """W warm-up steps, then K steps each bracketed by CUDA events (L2 flushed before each)."""
    import ctypes
    import torch
    from paper_1701_01189_b200 import _lib

    lib = _lib.load()
    for _ in range(warmup):
        flush()
        run.step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    stage = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    for st_ in stage:  # torch creates the cudaEvent lazily: force it before taking the handle
        for e in st_:
            e.record()
    handles = [(ctypes.c_void_p * 4)(*[e.cuda_event for e in st]) for st in stage]
    launches0 = lib.ms_launch_count()
    torch.cuda.synchronize()
    for i in range(steps):
        flush()
        if stage_events:
            lib.ms_set_stage_events(handles[i])
        ev[i][0].record()
        run.step()
        ev[i][1].record()
        lib.ms_set_stage_events(None)
    torch.cuda.synchronize()
    launches = lib.ms_launch_count() - launches0
    times = [a.elapsed_time(b) for a, b in ev]
    st = None
    if stage_events and run.bucket is not None:
        st = {
            "prescan": sum(s[0].elapsed_time(s[1]) for s in stage) / steps,
            "scan": sum(s[1].elapsed_time(s[2]) for s in stage) / steps,
            "postscan": sum(s[2].elapsed_time(s[3]) for s in stage) / steps,
        }
    return times, st, launches


def e2e_steps(run: Runner, steps: int, warmup: int):
    """Same metric through the public API with HOST buffers: pinned H2D of the inputs, the
    multisplit / sort, D2H of the outputs (and offsets), all inside the timed region."""
    import torch
    n = run.n
    if run.wl["kind"] == "sssp":  # H2D of the CSR graph, D2H of the distances
        hosts = [torch.from_numpy(a.view("int32")).pin_memory() for a in run.graph_host]
        devs = [torch.empty_like(x, device=run.rp.device) for x in hosts]
        dh = torch.empty(run.dist.numel(), dtype=torch.int32).pin_memory()

        def one_s():
            for d_, h_ in zip(devs, hosts):
                d_.copy_(h_, non_blocking=True)
            run.ms.sssp(devs[0], devs[1], devs[2], 0, delta=run.wl["delta"], buckets=run.m, out=run.dist,
                        workspace=run.ws)
            dh.copy_(run.dist, non_blocking=True)

        for _ in range(max(1, warmup)):
            one_s()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            one_s()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps, sum(4 * h.numel() for h in hosts), 4 * dh.numel()
    if run.wl["kind"].startswith("hist"):  # H2D of the samples, D2H of the m counts
        xh = run.samples.cpu().pin_memory()
        ch = torch.empty(run.m, dtype=torch.int32).pin_memory()
        xd = torch.empty_like(run.samples)

        def one_h():
            xd.copy_(xh, non_blocking=True)
            if run.wl["kind"] == "hist_even":
                run.ms.histogram_even(xd, run.m, 0.0, 1024.0, out=run.counts)
            else:
                run.ms.histogram_range(xd, run.splitters, out=run.counts)
            ch.copy_(run.counts, non_blocking=True)

        for _ in range(max(1, warmup)):
            one_h()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            one_h()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps, 4 * n, 4 * run.m
    kh = run.keys.cpu().pin_memory()
    vh = run.vals.cpu().pin_memory() if run.vals is not None else None
    h2d = 4 * n * (2 if vh is not None else 1)
    d2h = 4 * n * (2 if vh is not None else 1) + (4 * (run.m + 1) if run.bucket is not None else 0)
    if run.world > 1:  # registered output windows: one buffer set, steps in sequence
        koh = torch.empty(n, dtype=torch.int32).pin_memory()
        voh = torch.empty(n, dtype=torch.int32).pin_memory() if vh is not None else None
        kd = torch.empty_like(run.keys)
        vd = torch.empty_like(run.vals) if run.vals is not None else None

        def one():
            kd.copy_(kh, non_blocking=True)
            if vd is not None:
                vd.copy_(vh, non_blocking=True)
            saved = run.vals
            run.vals = vd
            run.step(keys=kd)
            run.vals = saved
            koh.copy_(run.ko, non_blocking=True)
            if voh is not None:
                voh.copy_(run.vo, non_blocking=True)

        for _ in range(max(1, warmup)):
            one()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            one()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps, h2d, d2h
    # one GPU: batches stream through the public API as an application would run
    # them -- step i's upload, its multisplit and step i-1's download overlap on
    # three streams (double-buffered device and pinned host buffers); every
    # step still copies its inputs in and its outputs (and offsets) out
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    pairs = vh is not None
    kd = [torch.empty_like(run.keys) for _ in range(2)]
    vd = [torch.empty_like(run.vals) for _ in range(2)] if pairs else [None, None]
    ko = [torch.empty_like(run.keys) for _ in range(2)]
    vo = [torch.empty_like(run.vals) for _ in range(2)] if pairs else [None, None]
    off = [torch.empty(run.m + 1, dtype=torch.int32, device=run.keys.device) for _ in range(2)]
    koh = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(2)]
    voh = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(2)] if pairs else [None, None]
    offh = [torch.empty(run.m + 1, dtype=torch.int32).pin_memory() for _ in range(2)]

    def batch(total):
        ev_comp, ev_out = [], []
        start = torch.cuda.Event(enable_timing=True)
        start.record(comp)
        s_in.wait_event(start)
        s_out.wait_event(start)
        for i in range(total):
            b = i % 2
            e_in = torch.cuda.Event()
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(ev_comp[i - 2])  # kd[b] read by step i-2
                kd[b].copy_(kh, non_blocking=True)
                if pairs:
                    vd[b].copy_(vh, non_blocking=True)
                e_in.record(s_in)
            comp.wait_event(e_in)
            if i >= 2:
                comp.wait_event(ev_out[i - 2])  # ko[b] downloaded by step i-2
            if run.bucket is None:
                run.ms.radix_sort(kd[b], vd[b], bits_per_pass=run.wl.get("bits", 8), out_keys=ko[b],
                                  out_values=vo[b], workspace=run.ws)
            else:
                run.ms.multisplit(kd[b], vd[b], bucket=run.bucket, out_keys=ko[b], out_values=vo[b],
                                  out_offsets=off[b], workspace=run.ws)
            e_c = torch.cuda.Event()
            e_c.record(comp)
            ev_comp.append(e_c)
            e_o = torch.cuda.Event()
            with torch.cuda.stream(s_out):
                s_out.wait_event(e_c)
                koh[b].copy_(ko[b], non_blocking=True)
                if pairs:
                    voh[b].copy_(vo[b], non_blocking=True)
                if run.bucket is not None:
                    offh[b].copy_(off[b], non_blocking=True)
                e_o.record(s_out)
            ev_out.append(e_o)
        comp.wait_event(ev_out[-1])
        end = torch.cuda.Event(enable_timing=True)
        end.record(comp)
        torch.cuda.synchronize()
        return start.elapsed_time(end) / total

    batch(max(2, warmup))
    t = batch(steps)
    # the streamed result equals the device-timed path's (same inputs)
    last = (steps - 1) % 2
    e2e_steps.parity = bool(torch.equal(koh[last], run.ko.cpu()) and
                            (not pairs or torch.equal(voh[last], run.vo.cpu())))
    return t, h2d, d2h


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = WORKLOADS[args.workload]
    m = args.m or wl["m"]
    hbm, peak_src = load_peaks()
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    from gen import device as gdev
    flush = lambda: gdev.flush_(scratch)  # noqa: E731

    if world > 1 and wl["kind"] == "sort":
        raise SystemExit("the sort workloads run on one GPU")
    run = Runner(wl, m, dev, rank, world)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local_rank) as clk:
        # the timed steps carry no stage events (events between kernels would
        # serialize the programmatic dependent launches); a separate pass below
        # records the per-stage breakdown for the roofline of the postscan
        times, _, launches = time_steps(run, args.steps, args.warmup, flush, stage_events=False)
        stages = None
        if world == 1:
            _, stages, _ = time_steps(run, max(3, args.steps // 2), 1, flush, stage_events=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_step = sum(times) / len(times)
    if world > 1:  # max over ranks of the device-timed step
        t = torch.tensor([ms_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    n = run.n
    uscale = 1e6 if wl["unit"] == "MTEPS" else 1e9
    value = n * world / (ms_step * 1e-3) / uscale  # all ranks' elements / max-over-ranks step time
    # dominant kernel = KF (kf_fused); algorithmic bytes per launch: read + write of keys (+ values)
    roofline = None
    if wl["kind"].startswith("hist"):  # one kernel (kh_histogram) + a counts memset
        achieved = 4 * n / (ms_step * 1e-3) / 1e9
        roofline = {"kernel": "kh_histogram (warp-private smem counts + one global atomic per CTA and bucket)",
                    "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(achieved / hbm, 4), "traffic": load_traffic(f"{args.workload}_m{m}"),
                    "alg_bytes_per_launch": 4 * n, "peak_source": peak_src}
    elif stages is not None:
        ks_bytes = n * (16 if wl["pairs"] else 8)
        achieved = ks_bytes / (stages["postscan"] * 1e-3) / 1e9
        kname = kernel_name(m if wl["kind"] != "sort" else 1 << wl.get("bits", 8))
        roofline = {"kernel": kname, "bound": "hbm", "achieved": round(achieved, 1),
                    "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                    "traffic": load_traffic(f"{args.workload}_m{m}"),
                    "alg_bytes_per_launch": ks_bytes, "peak_source": peak_src,
                    "stage_ms": {k: round(v, 5) for k, v in stages.items()}}
    whole_frac = value * uscale / world * wl["bpe"] / (hbm * 1e9)
    nominal_frac = value * uscale / world * wl["bpe"] / (NOMINAL_HBM_GBS * 1e9)
    e2e_ms, h2d, d2h = e2e_steps(run, max(3, args.steps // 4), 2)
    out = {
        "metric": metric_name(wl, args.workload, m),
        "value": round(value, 3), "unit": wl["unit"], "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "ms_per_step_median": round(statistics.median(times), 5), "ms_per_step_min": round(min(times), 5),
        "higher_is_better": True,
        "scaling": "strong" if wl.get("strong") else "weak", "vs_baseline": None, "dtype": "f32" if wl["kind"].startswith("hist") else "u32",
        "data": "synthetic (seeded counter-based generator)",
        "config": {"workload": wl["desc"], "n_per_rank": n, "n_total": n * world, "m": m, "bucket": wl["kind"],
                   "pairs": wl["pairs"], "l2": "flushed before every timed step (512 MiB write)",
                   "parallelism": (f"sharded{world} (libms: NCCL all-gather of counts + fused NVLink peer-store "
                                   f"scatter KP)" if world > 1 else "single")},
        "hbm_roofline_frac_whole_op": round(whole_frac, 4),
        "hbm_roofline_frac_whole_op_nominal_8tbs": round(nominal_frac, 4),
        "roofline": roofline,
        "e2e": {"value": round(n * world / (e2e_ms * 1e-3) / uscale, 3), "unit": wl["unit"],
                "matches_device_path": getattr(e2e_steps, "parity", None),
                "how": ("public API with pinned host buffers; per step H2D of the inputs, the call, D2H of the "
                        "outputs and offsets; steps overlap on three streams (double-buffered)" if world == 1 else
                        "public API with pinned host buffers; per step H2D, the sharded call, D2H, in sequence"),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_sweep:
        out["sweep"] = sweep(args, dev, flush, hbm)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl, m)
        out["cpu_parallel"] = cpu_parallel(wl, m)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sweep(args, dev, flush, hbm):
    """Per-m throughput table (BASELINE.md section 2 layout), a few steps each: keys and
    pairs at every m of the metric (2..256, configs[1] size), configs[2] identity and
    radix digits (uniform and 90 % skew), configs[3] sorts, configs[0] latency, f2."""
    import torch
    res = {}
    cases = [("ms_keys", m) for m in (2, 4, 8, 16, 32, 64, 128, 256)] + \
            [("ms_pairs", m) for m in (2, 4, 8, 16, 32, 64, 128, 256)] + \
            [("ms_pairs_c3", 64), ("ms_pairs_c3", 128), ("ms_pairs_c3", 256), ("ms_pairs_c3_skew", 256),
             ("ms_pairs_c3_radix", 64), ("ms_pairs_c3_radix", 128), ("ms_pairs_c3_radix", 256),
             ("ms_pairs_c3_radix_skew", 256),
             ("sort_keys", 256), ("sort_pairs", 256), ("sort_keys_passes", 256), ("sort_pairs_passes", 256),
             ("sort_keys_r5", 32), ("sort_pairs_r5", 32),
             ("ms_keys_os", 2), ("ms_keys_os", 32), ("ms_keys_os", 256), ("ms_pairs_os", 32), ("ms_pairs_os", 256),
             ("hist_even", 2), ("hist_even", 256), ("hist_range", 2), ("hist_range", 256),
             ("ms_keys_spl", 32), ("ms_keys_spl", 256), ("ms_pairs_spl", 256),
             ("ms_keys_large", 1024), ("ms_keys_large", 65536), ("ms_pairs_large", 4096),
             ("sssp_rmat", 10)]
    for name, m in cases:
        wl = WORKLOADS[name]
        run = Runner(wl, m, dev)
        steps = 5 if wl["kind"] == "sort" else 10
        times, _, _ = time_steps(run, steps, 3, flush, stage_events=False)
        _, stages, _ = time_steps(run, 3, 1, flush, stage_events=True)
        t = sum(times) / len(times)
        us = 1e6 if wl["unit"] == "MTEPS" else 1e9
        rate = run.n / (t * 1e-3) / us
        e = {"value": round(rate, 2), "unit": wl["unit"], "ms": round(t, 4),
             "hbm_frac": round(rate * us * wl["bpe"] / (hbm * 1e9), 3),
             "hbm_frac_nominal": round(rate * us * wl["bpe"] / (NOMINAL_HBM_GBS * 1e9), 3)}
        if "bpe_f1" in wl:  # against the one-pass sort's own bound (36 / 68 B)
            e["hbm_frac_f1"] = round(rate * us * wl["bpe_f1"] / (hbm * 1e9), 3)
        if wl["kind"] == "sssp":
            e["iterations"] = run.sssp_stats()["iterations"]
        if stages:
            e["stage_ms"] = {k: round(v, 4) for k, v in stages.items()}
            e["kf_frac"] = round(wl["n"] * (16 if wl["pairs"] else 8) / (stages["postscan"] * 1e-3) / 1e9 / hbm, 3)
        res[f"{name}_m{m}"] = e
        del run
        torch.cuda.empty_cache()
    res["c1_latency"] = c1_latency(dev)
    return res


def c1_latency(dev):
    """configs[0]: n = 2^10 keys, m = 2 delta buckets -- microseconds per call through the
    public API (one launch, latency-bound), back to back and replayed from a CUDA graph,
    next to the CPU stable counting sort (the oracle) on the same keys."""
    import numpy as np
    import torch
    import oracle
    import paper_1701_01189_b200 as ms
    from gen import inputs as gen
    n, m = 1 << 10, 2
    fn = oracle.delta(m)
    kh = gen.keys(n, SEED, kind=gen.DELTA, m=m, delta=fn.delta)
    k = torch.from_numpy(kh.view(np.int32)).to(dev)
    ko = torch.empty_like(k)
    off = torch.empty(m + 1, dtype=torch.int32, device=dev)
    ws = torch.empty(max(1, ms.workspace_size(n, m, False)), dtype=torch.uint8, device=dev)
    b = ms.Delta(m)
    call = lambda: ms.multisplit(k, None, bucket=b, out_keys=ko, out_offsets=off, workspace=ws)  # noqa: E731
    for _ in range(20):
        call()
    torch.cuda.synchronize()
    reps = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    us_call = e0.elapsed_time(e1) * 1e3 / reps
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            call()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps // 10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us_graph = e0.elapsed_time(e1) * 1e3 / reps
    ok = np.array_equal(ko.cpu().numpy().view(np.uint32), oracle.multisplit(kh, fn)[0])
    t0 = time.perf_counter()
    for _ in range(200):
        oracle.multisplit(kh, fn)
    us_cpu = (time.perf_counter() - t0) * 1e6 / 200
    return {"unit": "us/call", "gpu_us_per_call": round(us_call, 3), "gpu_us_per_call_cuda_graph": round(us_graph, 3),
            "cpu_oracle_us_per_call": round(us_cpu, 3), "parity": bool(ok),
            "note": "n=2^10, m=2; the oracle time includes the ctypes call from Python"}


# --------------------------------------------------------------------------- oracle (CPU) arm
def _oracle_sample(wl, m, n_sample):
    import numpy as np
    import oracle
    from gen import inputs as gen
    kind = wl["kind"]
    dist = {"skew": gen.DIST_SKEW}.get(wl.get("dist"), gen.DIST_UNIFORM)
    if kind == "delta":
        fn = oracle.delta(m)
        k = gen.keys(n_sample, SEED, kind=gen.DELTA, m=m, delta=fn.delta, dist=dist, alpha=0.1)
    elif kind == "identity":
        fn = oracle.identity(m)
        k = gen.keys(n_sample, SEED, kind=gen.IDENTITY, m=m, dist=dist, alpha=0.1)
    elif kind == "splitters":
        r = np.random.default_rng(SEED + m)
        fn = oracle.splitters(np.sort(r.choice(1 << 32, size=m - 1, replace=False).astype(np.uint64)))
        k = gen.keys(n_sample, SEED)
    elif kind == "sssp":  # the R-MAT graph at the workload's scale, or 2 smaller for a bounded sample
        from gen.graphs import rmat_csr
        V, rp, col, w = rmat_csr(wl["scale"] - (2 if n_sample < (1 << 25) else 0), wl["ef"], SEED, undirected=True)
        f = lambda: oracle.sssp(rp, col, w, 0)  # noqa: E731
        f.units = int(col.size)
        return f
    else:
        fn = None
        k = gen.keys(n_sample, SEED)
    v = gen.values(n_sample, SEED, parity=False) if wl["pairs"] else None
    if kind == "hist_even":
        x = gen.floats(n_sample, SEED)
        return lambda: oracle.histogram_even(x, m, 0.0, 1024.0)
    if kind == "hist_range":
        x = gen.floats(n_sample, SEED)
        spl = gen.splitters(m, SEED)
        return lambda: oracle.histogram_range(x, spl)
    if fn is None:
        return lambda: oracle.radix_sort(k, v)
    return lambda: oracle.multisplit(k, fn, v)


def cpu_baseline(wl, m, budget_s: float = 12.0):
    """The oracle as it stands (single-threaded C) on the host, bounded sample."""
    n_sample = min(wl["n"], 1 << 25) if wl["kind"] not in ("sort", "sssp") else (1 << 22 if wl["kind"] == "sort" else 1 << 25)
    f = _oracle_sample(wl, m, n_sample)
    n_sample = getattr(f, "units", n_sample)
    us = 1e6 if wl["unit"] == "MTEPS" else 1e9
    f()
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        f()
        reps += 1
    dt = (time.perf_counter() - t0) / reps
    return {"value": round(n_sample / dt / us, 4), "unit": wl["unit"], "cores": 1, "kind": "oracle",
            "sample": f"{reps} x {n_sample} elements of the same workload (seed {SEED})",
            "host_cores_available": len(os.sched_getaffinity(0))}


def cpu_parallel(wl, m, budget_s: float = 6.0):
    """The paper's {local, global, local} multisplit on ALL host cores (baseline/, C with
    pthreads) on a bounded sample of the workload: context for the GPU rate."""
    import numpy as np
    import baseline
    import oracle
    from gen import inputs as gen
    cores = len(os.sched_getaffinity(0))
    kind = wl["kind"]
    n_sample = min(wl["n"], 1 << 25)
    if kind.startswith("hist") or kind in ("sssp", "splitters") or m > 256:
        return None
    if kind == "sort":
        k = gen.keys(n_sample, SEED)
        v = gen.values(n_sample, SEED, parity=False) if wl["pairs"] else None
        f = lambda: baseline.radix_sort(k, v, wl.get("bits", 8), cores)  # noqa: E731
    else:
        if kind == "delta":
            fn = oracle.delta(m)
            k = gen.keys(n_sample, SEED, kind=gen.DELTA, m=m, delta=fn.delta)
            kw = dict(delta=fn.delta)
        else:  # identity / radix: digits of the low bits
            bits = max(1, (m - 1).bit_length())
            k = gen.keys(n_sample, SEED, kind=gen.RADIX, m=1 << bits, shift=0, bits=bits)
            kw = dict(bits=bits)
        v = gen.values(n_sample, SEED, parity=False) if wl["pairs"] else None
        f = lambda: baseline.multisplit(k, v, m if kind == "delta" else 1 << kw.get("bits", 1), threads=cores, **kw)  # noqa: E731
    f()
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        f()
        reps += 1
    dt = (time.perf_counter() - t0) / reps
    return {"value": round(n_sample / dt / 1e9, 4), "unit": wl["unit"], "cores": cores, "kind": "parallel C (pthreads)",
            "sample": f"{reps} x {n_sample} elements of the same workload (seed {SEED})"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    m = args.m or wl["m"]
    n_sample = min(wl["n"], 1 << 24) if wl["kind"] != "sort" else (1 << 21)
    f = _oracle_sample(wl, m, n_sample)
    n_sample = getattr(f, "units", n_sample)
    for _ in range(args.warmup):
        f()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    dt = sum(ts) / len(ts)
    value = n_sample / dt / (1e6 if wl["unit"] == "MTEPS" else 1e9)
    out = {"impl": "reference",
           "metric": metric_name(wl, args.workload, m),
           "value": round(value, 4), "unit": wl["unit"], "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32" if wl["kind"].startswith("hist") else "u32", "data": "synthetic (seeded counter-based generator)",
           "config": {"workload": wl["desc"], "n": wl["n"], "m": m, "bucket": wl["kind"], "pairs": wl["pairs"]},
           "cpu_baseline": {"value": round(value, 4), "unit": wl["unit"], "cores": 1, "kind": "oracle",
                            "sample": f"each step: {n_sample} elements of the workload (seed {SEED})"},
           "e2e": {"value": round(value, 4), "unit": wl["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)  # the paper averages 50 trials
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="ms_keys")
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not under torchrun: launch N ranks (one process per GPU) ourselves
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
