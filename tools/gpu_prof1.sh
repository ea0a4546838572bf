#!/bin/bash
# Full ncu capture of one kernel (regex) on the bench workload.
# usage: gpurun -- bash tools/gpu_prof1.sh <tag> <kernel-regex> [skip]
tag=$1; k=$2; skip=${3:-2}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $skip -c 1 \
    -o $out/prof_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/ncu_$k.log 2>&1
tail -3 $out/ncu_$k.log
