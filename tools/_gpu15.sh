#!/bin/bash
out=gpurun_out/r1y; mkdir -p $out
BMG_TIMELINE=1 timeout 300 python tools/e2e_probe.py shard16k > $out/probe16k.log 2>&1
python tools/h2d_probe.py > $out/h2d.log 2>&1
grep -n "upload\|row 0 start\|^py" $out/probe16k.log | tail -32; cat $out/h2d.log
