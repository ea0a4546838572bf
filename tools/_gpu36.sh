#!/bin/bash
out=gpurun_out/r1ay; mkdir -p $out
for k in codes_tma_kernel tables_fused_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 \
      -o $out/prof_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/ncu_$k.log 2>&1
done
ls $out
