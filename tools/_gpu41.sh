#!/bin/bash
out=gpurun_out/r1bh; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_match.py tests/test_gpu_engine.py -x -q > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
tail -2 $out/pytest.log
bash tools/_ab.sh r1bh base old base
for v in base old; do lib=paper_2505_22089_b200/libbmg.so; [ $v != base ] && lib=paper_2505_22089_b200/libbmg_$v.so
BMG_LIBBMG=$PWD/$lib timeout 600 python bench.py --config shard16k --steps 3 --warmup 2 --no-cpu-baseline > $out/b16_$v.json 2>/dev/null
python - $out/b16_$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], 'shard16k', round(d['value']), round(d['e2e']['value']), round(d['kernel_ms_per_step']['match'],2))
PY
done
