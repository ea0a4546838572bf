#!/bin/bash
# VLAD encoder on the box: GPU tests, timing probe, ncu of the assign kernel.
tag=${1:-vlad}; out=gpurun_out/$tag; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_retrieval.py -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 600 python tests/probes/vlad_probe.py 500 32 > $out/probe.json 2> $out/probe.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vlad -c 4 -o $out/prof_vlad python tests/probes/vlad_probe.py 16 2 > $out/ncu.log 2>&1
tail -3 $out/pytest.log; cat $out/probe.json; tail -3 $out/probe.err
