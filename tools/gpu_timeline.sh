#!/bin/bash
# Per-row event timeline of the e2e execute_plan on the bench workload.
# usage: gpurun -- bash tools/gpu_timeline.sh TAG [config] [pageable]
tag=$1; cfg=${2:-strip500}; src=${3:-pinned}
out=gpurun_out/$tag; mkdir -p $out
BMG_TIMELINE=1 timeout 600 python tools/e2e_probe.py $cfg 4 $src > $out/timeline_${cfg}_$src.log 2>&1
grep -v 'upload [0-9]*[13579] ' $out/timeline_${cfg}_$src.log | tail -24
