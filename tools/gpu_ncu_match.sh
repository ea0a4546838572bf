#!/bin/bash
# Full ncu capture (source-level) of match_kernel on the block32 workload.
# usage: gpurun -- bash tools/gpu_ncu_match.sh <tag> [config]
tag=$1; cfg=${2:-block32}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-match_kernel} -s 2 -c 1 \
    -o $out/prof_match python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --no-files > $out/ncu_match.log 2>&1
tail -3 $out/ncu_match.log
