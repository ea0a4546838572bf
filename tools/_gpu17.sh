#!/bin/bash
out=gpurun_out/r1aa; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q > $out/pytest_engine.log 2>&1; echo "rc=$?" >> $out/pytest_engine.log
tail -3 $out/pytest_engine.log
BMG_TIMELINE=1 timeout 300 python tools/e2e_probe.py block32 > $out/probe32.log 2>&1
grep -v "upload [0-9]" $out/probe32.log | tail -22
