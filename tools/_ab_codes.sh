t=${1:-abc}; shift
mkdir -p gpurun_out/$t
for v in "$@"; do
  lib=paper_2505_22089_b200/libbmg_$v.so; [ "$v" = base ] && lib=paper_2505_22089_b200/libbmg.so
  BMG_LIBBMG=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:codes_kernel -c 40 --csv --log-file gpurun_out/$t/l_$v.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  python - "$t" "$v" <<'PY'
import sys, csv, io
t, v = sys.argv[1], sys.argv[2]
txt = open(f"gpurun_out/{t}/l_{v}.csv").read(); txt = txt[txt.find('"ID"'):]
ms = [float(r["Metric Value"].replace(",", "")) / 1e6 for r in csv.DictReader(io.StringIO(txt)) if r.get("Metric Name") == "gpu__time_duration.sum"]
print(f"{v:10s} codes launches {len(ms)} mean {sum(ms)/max(len(ms),1):.4f} ms  max {max(ms):.4f}")
PY
done
