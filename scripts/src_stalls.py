"""Per-CUDA-source-line stall samples from an ncu report (-lineinfo, --import-source on):
python src_stalls.py rep.ncu-rep [top] -> the lines with the most warp-stall samples."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the CSV may hold several files, each with its own header row
hdr = None
items = []
cur_file = ""
for r in rows:
    if not r:
        continue
    if "Source" in r and ("Warp Stall Sampling (All Samples)" in r):
        hdr = r
        continue
    if hdr is None:
        if len(r) == 1:
            cur_file = r[0]
        continue
    if len(r) != len(hdr):
        if len(r) == 1:
            cur_file = r[0]
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    if s:
        items.append((s, cur_file[-40:], d.get("#", d.get("Line", "")), d["Source"].strip()[:110]))
tot = sum(i[0] for i in items)
print("total samples", tot)
for s, f, ln, src in sorted(items, reverse=True)[:top]:
    print(f"{s:6d} {100.0 * s / max(tot, 1):5.1f}%  {f}:{ln}  {src}")
