#!/bin/bash
out=gpurun_out/r1v; mkdir -p $out
python tools/exact_probe.py 8192 16 >> $out/exact.log 2>&1
python tools/exact_probe.py 2000 16 >> $out/exact.log 2>&1
python tools/exact_probe.py 16384 8 >> $out/exact.log 2>&1
bash tools/gpu_prof1.sh r1v match_kernel 2
cat $out/exact.log
