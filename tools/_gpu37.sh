#!/bin/bash
out=gpurun_out/r1bf; mkdir -p $out
BMG_TIMELINE=1 timeout 300 python tools/e2e_probe.py block32 > $out/probe32.log 2>&1
grep -v "upload [0-9]" $out/probe32.log | tail -13
BMG_TIMELINE=1 timeout 300 python tools/e2e_probe.py strip500 > $out/probe500.log 2>&1
grep -v "upload [0-9]" $out/probe500.log | tail -19
