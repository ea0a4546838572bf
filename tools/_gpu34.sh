#!/bin/bash
out=gpurun_out/r1aw; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_mean.py tests/test_gpu_engine.py tests/test_gpu_codes.py -x -q > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
tail -2 $out/pytest.log
for c in block32 shard16k; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_$c.json 2> $out/bench_$c.err
python - $out/bench_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d['config']['workload'][:8], round(d['value']), round(d['e2e']['value']), {k:round(v,3) for k,v in d['kernel_ms_per_step'].items()})
PY
done
