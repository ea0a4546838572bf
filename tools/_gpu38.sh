#!/bin/bash
out=gpurun_out/r1be; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
tail -2 $out/pytest.log
for c in block32 strip500 shard16k; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_$c.json 2> $out/bench_$c.err
python - $out/bench_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d['config']['workload'][:8], round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), {k:round(v,3) for k,v in d['kernel_ms_per_step'].items()}, d['results_consistent_e2e_vs_resident'])
PY
done
grep -v "upload [0-9]" $out/probe32.log | tail -13


BMG_TIMELINE=1 timeout 300 python tools/e2e_probe.py block32 > $out/probe32.log 2>&1; grep -v "upload [0-9]" $out/probe32.log | tail -13
