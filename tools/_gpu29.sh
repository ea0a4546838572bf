#!/bin/bash
out=gpurun_out/r1ar; mkdir -p $out
timeout 1500 python tools/sweep.py --out $out/r1_sweep.md > $out/sweep.log 2>&1; echo "rc=$?" >> $out/sweep.log
tail -3 $out/sweep.log; cat $out/r1_sweep.md
