#!/bin/bash
out=gpurun_out/r1bg; mkdir -p $out
for v in base q512 q256; do lib=paper_2505_22089_b200/libbmg.so; [ $v != base ] && lib=paper_2505_22089_b200/libbmg_$v.so
for c in block32 strip500; do BMG_LIBBMG=$PWD/$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_${c}_$v.json 2> $out/bench_${c}_$v.err
python - $out/bench_${c}_$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], d['config']['workload'][:8], round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), round(d['kernel_ms_per_step']['match'],3))
PY
done; done
