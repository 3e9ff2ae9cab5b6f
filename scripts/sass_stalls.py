"""Per-instruction stall attribution from an ncu SASS source CSV:
python sass_stalls.py rep.ncu-rep [reason ...] -> top instructions per stall reason."""
import csv, io, subprocess, sys
rep = sys.argv[1]
reasons = sys.argv[2:] or ["stall_short_sb", "stall_long_sb", "stall_barrier", "stall_wait", "stall_mio"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]; rows = r[2:]
iS = h.index("Source"); iE = h.index("Instructions Executed")
for rs in reasons:
    ix = h.index(rs)
    tot = sum(int(x[ix] or 0) for x in rows)
    print(f"== {rs} total {tot}")
    top = sorted(range(len(rows)), key=lambda k: -int(rows[k][ix] or 0))[:8]
    for k in top:
        x = rows[k]
        print(f"  {k:5d} {int(x[ix] or 0):6d} exec {x[iE]:>8s}  {x[iS][:80]}  | prev: {rows[k-1][iS][:50]}")
