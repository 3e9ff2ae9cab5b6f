"""Summarise an .ncu-rep: key metrics + SASS opcode histogram + top stall reasons."""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Executed Instructions",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Block Limit Registers", "Block Limit Shared Mem",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Grid Size", "Waves Per SM"]
for r in det[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
rh, ru, rv = raw[0], raw[1], raw[2]
for k, u, v in zip(rh, ru, rv):
    if any(s in k for s in ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__pcsamp_warps_issue_stalled"]) \
            and not k.endswith("_not_issued") and v not in ("0", ""):
        print(f"{k:70s} {v:>16s} {u}")
sass = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
hdr = sass[1]; data = sass[2:]
ix = hdr.index("Instructions Executed"); isamp = hdr.index("Warp Stall Sampling (All Samples)")
c, s = Counter(), Counter()
for r in data:
    if not r[1]: continue
    toks = r[1].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    c[op] += int(r[ix] or 0); s[op] += int(r[isamp] or 0)
tot = sum(c.values())
n = float(sys.argv[2]) if len(sys.argv) > 2 else None
print("total warp instructions", tot, ("thread-instr/elem %.1f" % (tot * 32 / n)) if n else "")
for op, v in c.most_common(24):
    print(f"  {op:10s} {v:>12d} {('%.2f' % (v*32/n)) if n else '':>7s}  samples {s[op]}")
