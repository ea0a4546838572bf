# A/B of libbmg variants on the bench workload: resident value + ncu match time
t=${1:-ab}; shift
mkdir -p gpurun_out/$t
for v in "$@"; do
  lib=paper_2505_22089_b200/libbmg_$v.so; [ "$v" = base ] && lib=paper_2505_22089_b200/libbmg.so
  BMG_LIBBMG=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$t/bench_$v.json 2>/dev/null
  BMG_LIBBMG=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${ABK:-match} -c 40 --csv --log-file gpurun_out/$t/l_$v.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  python - "$t" "$v" <<'PY'
import json, sys, csv, io
t, v = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/{t}/bench_{v}.json"))
txt = open(f"gpurun_out/{t}/l_{v}.csv").read(); txt = txt[txt.find('"ID"'):]
ms = [float(r["Metric Value"].replace(",", "")) / 1e6 for r in csv.DictReader(io.StringIO(txt)) if r.get("Metric Name") == "gpu__time_duration.sum"]
print(f"{v:10s} value {d['value']:8.0f} e2e {d['e2e']['value']:8.0f} step {d['ms_per_step']:.3f} ms  match launches {len(ms)} mean {sum(ms)/max(len(ms),1):.3f} ms")
PY
done
