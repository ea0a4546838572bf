#!/bin/bash
# Sanitizers over the VLAD tests + one ncu --set full of each VLAD kernel at 64 images.
tag=${1:-vladprof}; out=gpurun_out/$tag; mkdir -p $out
SAN_SEL="tests/test_gpu_retrieval.py" bash tools/sanitize.sh $tag
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vlad -c 6 -o $out/prof_vlad64 \
  python tests/probes/vlad_probe.py 64 2 > $out/ncu64.log 2>&1
timeout 600 python tests/probes/vlad_probe.py 500 32 > $out/probe.json 2> $out/probe.err
cat $out/probe.json
