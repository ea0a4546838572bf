#!/bin/bash
out=gpurun_out/r1ah; mkdir -p $out
timeout 900 python tools/io_bench.py 64 16384 $out/io.json > $out/io.log 2>&1; tail -2 $out/io.log
