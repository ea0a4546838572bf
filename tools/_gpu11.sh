#!/bin/bash
out=gpurun_out/r1u; mkdir -p $out
for v in base lk4; do lib=paper_2505_22089_b200/libbmg.so; [ $v != base ] && lib=paper_2505_22089_b200/libbmg_$v.so
  BMG_LIBBMG=$PWD/$lib python tools/exact_probe.py 8192 16 >> $out/exact.log 2>&1
  BMG_LIBBMG=$PWD/$lib python tools/exact_probe.py 2000 16 >> $out/exact.log 2>&1
  BMG_LIBBMG=$PWD/$lib python tools/exact_probe.py 16384 8 >> $out/exact.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
bash tools/_ab.sh r1u base lk4
tail -2 $out/pytest_gpu.log; cat $out/exact.log
