#!/bin/bash
out=gpurun_out/r1at; mkdir -p $out
timeout 600 python bench.py --config pair1 --steps 20 --warmup 5 > $out/bench_pair1.json 2> $out/bench_pair1.err; echo "rc=$?"
tail -3 $out/bench_pair1.err
python - $out/bench_pair1.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['e2e']['ms_per_step'], d['cpu_baseline'], {k:round(v,3) for k,v in d['kernel_ms_per_step'].items()}, d['roofline']['frac'])
PY
