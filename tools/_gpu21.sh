#!/bin/bash
out=gpurun_out/r1ag; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
timeout 900 python tools/io_bench.py 64 16384 $out/io.json > $out/io.log 2>&1; tail -2 $out/io.log
