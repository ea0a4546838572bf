"""Instructions executed per unit of work, per source line (in line order),
from an ncu report: python tools/ncu_byline.py REP UNITS [min_per_unit]"""
import csv, io, subprocess, sys
rep, units = sys.argv[1], float(sys.argv[2])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
iI = hdr.index("Instructions Executed"); iS = hdr.index("Warp Stall Sampling (All Samples)")
tot_s = 0; recs = []
for r in rows[1:]:
    if len(r) > max(iI, iS) and r[0]:
        try:
            recs.append((int(r[0]), int(r[iI] or 0), int(r[iS] or 0), r[1][:100]))
            tot_s += int(r[iS] or 0)
        except ValueError:
            pass
tot = sum(x[1] for x in recs)
print(f"total {tot/units:.1f} inst/unit")
for ln, ni, ns, src in sorted(recs):
    if ni / units >= thr or 100 * ns / max(tot_s, 1) >= 1.0:
        print(f"{ln:5d} {ni/units:7.1f} stall {100*ns/max(tot_s,1):5.1f}%  {src}")
