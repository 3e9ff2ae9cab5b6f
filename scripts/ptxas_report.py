"""Compile the kernel TUs with -Xptxas -v and print registers / spills per kernel."""
import os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1701_01189_b200 import build as b
srcs = sys.argv[1:] or ["ms_inst_deltashift.cu"]
for src in srcs:
    cmd = [b.NVCC, *b.ARCH, *b.FLAGS, "-Xptxas=-v", "-c", os.path.join(b.CSRC, src), "-o", "/tmp/x.o"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    cur = None
    for ln in r.stderr.splitlines():
        m = re.search(r"Compiling entry function '(\w+)'", ln)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            cur = cur.replace("ms::", "").replace("(ms::KfArgs, ms::BucketParams)", "")
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if m and cur:
            spill = f"spill {m.group(1)}/{m.group(2)}"
        m2 = re.search(r"Used (\d+) registers", ln)
        if m2 and cur:
            print(f"{cur[:70]:70s} regs {m2.group(1):>3s}  {spill}")
            cur = None
    if r.returncode:
        print(r.stderr[-2000:])
