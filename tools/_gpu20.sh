#!/bin/bash
out=gpurun_out/r1af; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
for v in 0; do
for c in block32 strip500 shard16k; do BMG_LOG_ZC=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_${c}_$v.json 2> $out/bench_${c}_$v.err; done
for c in block32 strip500 shard16k; do python - $out/bench_${c}_$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], d['config']['workload'][:10], round(d['value']), round(d['e2e']['value']), d['e2e']['step_ms'][:5], d['results_consistent_e2e_vs_resident'], d['kernel_ms_per_step'].get('compact'))
PY
done; done
