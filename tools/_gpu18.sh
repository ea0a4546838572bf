#!/bin/bash
out=gpurun_out/r1ac; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
for c in block32 strip500 shard16k; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_$c.json 2> $out/bench_$c.err; done
for c in block32 strip500 shard16k; do python - $out/bench_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d['config']['workload'][:10], round(d['value']), round(d['e2e']['value']), d['e2e']['step_ms'][:5], d['results_consistent_e2e_vs_resident'])
PY
done
BMG_TIMELINE=1 timeout 300 python tools/e2e_probe.py block32 > $out/probe32.log 2>&1
grep -v "upload [0-9]" $out/probe32.log | tail -12
