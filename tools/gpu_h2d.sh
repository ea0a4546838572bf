#!/bin/bash
tag=${1:-h2d}; out=gpurun_out/$tag; mkdir -p $out
timeout 300 python tools/h2d_probe.py > $out/h2d.log 2>&1
BMG_TIMELINE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-retrieval --no-files > $out/tl.json 2> $out/tl.err
cat $out/h2d.log; grep "bmg timeline" $out/tl.err | tail -40
