#!/bin/bash
out=gpurun_out/r1am; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_mean.py -x -q > $out/pytest_mean.log 2>&1; echo "rc=$?" >> $out/pytest_mean.log
tail -2 $out/pytest_mean.log
for v in base old; do lib=paper_2505_22089_b200/libbmg.so; [ $v = old ] && lib=paper_2505_22089_b200/libbmg_old.so
for c in block32 shard16k; do BMG_LIBBMG=$PWD/$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_${c}_$v.json 2> $out/bench_${c}_$v.err
python - $out/bench_${c}_$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], d['config']['workload'][:10], round(d['value']), round(d['e2e']['value']), {k:round(v,3) for k,v in d['kernel_ms_per_step'].items()})
PY
done; done
