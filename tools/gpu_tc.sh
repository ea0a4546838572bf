#!/bin/bash
tag=${1:-tc}; out=gpurun_out/$tag; mkdir -p $out
for v in base tc512; do
  lib=$PWD/paper_2505_22089_b200/libbmg.so; [ $v != base ] && lib=$PWD/paper_2505_22089_b200/libbmg_$v.so
  BMG_LIBBMG=$lib timeout 900 python -m pytest tests/test_gpu_codes.py tests/test_gpu_mean.py tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider > $out/pytest_$v.log 2>&1; echo "$v $(tail -1 $out/pytest_$v.log)"
done
bash tools/ab_libs.sh ${tag}_ab base tc512
for v in base tc512; do
  lib=$PWD/paper_2505_22089_b200/libbmg.so; [ $v != base ] && lib=$PWD/paper_2505_22089_b200/libbmg_$v.so
  python3 -c "
import json; d=json.loads(open('gpurun_out/${tag}_ab/strip500_$v.json').read().strip().splitlines()[-1]); print('$v', d['kernel_ms_per_step'])"
done
