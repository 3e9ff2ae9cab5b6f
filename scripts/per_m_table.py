"""Summarise gpurun_out/.../perm/*.csv (ncu --csv, one multisplit per run) into a
markdown table: per kernel of the last call, time, DRAM bytes vs algorithmic,
instructions per element, store sectors per request, smem bank conflicts."""
import csv, glob, os, sys, collections
d = sys.argv[1]
N = 1 << 25
rows_out = []
for f in sorted(glob.glob(os.path.join(d, "*.csv")), key=lambda p: (os.path.basename(p).split("_m")[0], int(p.split("_m")[-1][:-4]))):
    name = os.path.basename(f)[:-4]
    wl, m = name.rsplit("_m", 1)
    n = (1 << 27) if "c3" in wl else N
    pairs = "pairs" in wl
    lines = [l for l in open(f) if l.startswith('"')]
    rd = list(csv.reader(lines))
    if not rd:
        continue
    hdr = rd[0]
    per = collections.OrderedDict()
    for r in rd[1:]:
        x = dict(zip(hdr, r))
        key = (x["ID"], x["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("ms::", ""))
        per.setdefault(key, {})[x["Metric Name"]] = float(x["Metric Value"].replace(",", "") or 0)
    # the last call: the last occurrence of each kernel name
    last = collections.OrderedDict()
    for (i, k), v in per.items():
        last[k] = v
    for k, v in last.items():
        t = v.get("gpu__time_duration.sum", 0) / 1e3
        rdb, wrb = v.get("dram__bytes_read.sum", 0), v.get("dram__bytes_write.sum", 0)
        ins = v.get("smsp__inst_executed.sum", 0) * 32 / n
        sec, req = v.get("lts__t_sectors_srcunit_tex_op_write.sum", 0), v.get("lts__t_requests_srcunit_tex_op_write.sum", 0)
        bc = v.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 0) / n
        dp = v.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0)
        rows_out.append(f"| {wl} | {m} | {k} | {t:.1f} | {rdb/1e6:.0f} | {wrb/1e6:.0f} | {dp:.0f} | {ins:.1f} | {sec/req if req else 0:.2f} | {bc:.2f} |")
print("| workload | m | kernel | µs | DRAM read MB | DRAM write MB | DRAM % peak | thread-instr / element | L2 store sectors / request | smem bank conflicts / element |")
print("|---|---|---|---|---|---|---|---|---|---|")
print("\n".join(rows_out))
