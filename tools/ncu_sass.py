"""Hot SASS instructions of an ncu report, per unit of work:
python tools/ncu_sass.py REP UNITS [min_per_unit]"""
import csv, io, subprocess, sys
rep, units = sys.argv[1], float(sys.argv[2])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 3.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
iI = hdr.index("Instructions Executed"); iS = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
for r in rows[1:]:
    if len(r) > iI:
        try:
            ni = int(r[iI] or 0)
        except ValueError:
            continue
        if ni / units >= thr:
            print(f"{ni/units:6.1f} {int(r[iS] or 0):6d} {r[src][:90]}")
