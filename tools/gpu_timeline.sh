#!/bin/bash
# Per-row event timeline of the e2e execute_plan on the bench workload.
# usage: gpurun -- bash tools/gpu_timeline.sh TAG [config]
tag=$1; cfg=${2:-strip500}
out=gpurun_out/$tag; mkdir -p $out
BMG_TIMELINE=1 timeout 600 python tools/e2e_probe.py $cfg > $out/timeline_$cfg.log 2>&1
grep -v 'upload [0-9]' $out/timeline_$cfg.log | tail -60
