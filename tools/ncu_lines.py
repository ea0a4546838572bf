"""Per-source-line hot spots of an ncu report (instructions executed and stall
samples), from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
iI = hdr.index("Instructions Executed"); iS = hdr.index("Warp Stall Sampling (All Samples)")
agg = []
tot_i = tot_s = 0
for r in rows[1:]:
    if len(r) > max(iI, iS) and r[0]:  # a source line row (aggregated)
        try:
            ni = int(r[iI] or 0); ns = int(r[iS] or 0)
        except ValueError:
            continue
        agg.append((ni, ns, r[0], r[1][:110]))
        tot_i += ni; tot_s += ns
agg.sort(key=lambda x: -x[1])
print(f"total inst {tot_i:,}  stall samples {tot_s:,}")
for ni, ns, ln, src in agg[:top]:
    print(f"{ln:>5} inst {100*ni/max(tot_i,1):5.1f}%  stall {100*ns/max(tot_s,1):5.1f}%  {src}")
