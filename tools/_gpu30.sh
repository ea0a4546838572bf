#!/bin/bash
out=gpurun_out/r1as; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
tail -2 $out/pytest.log
for v in base old base; do lib=paper_2505_22089_b200/libbmg.so; [ $v = old ] && lib=paper_2505_22089_b200/libbmg_old.so
BMG_LIBBMG=$PWD/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_$v.json 2> $out/bench_$v.err
python - $out/bench_$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(d['value']), round(d['e2e']['value']), {k:round(v,3) for k,v in d['kernel_ms_per_step'].items()})
PY
done
