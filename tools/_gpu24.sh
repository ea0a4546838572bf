#!/bin/bash
out=gpurun_out/r1aj; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_codes.py -x -q > $out/pytest_codes.log 2>&1; echo "rc=$?" >> $out/pytest_codes.log
tail -15 $out/pytest_codes.log
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
for v in 0 1; do BMG_PROJECT_SIMT=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_$v.json 2> $out/bench_$v.err
python - $out/bench_$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('simt' if sys.argv[2]=='1' else 'tc  ', round(d['value']), round(d['e2e']['value']), {k:round(v,3) for k,v in d['kernel_ms_per_step'].items()}, d['results_consistent_e2e_vs_resident'])
PY
done
