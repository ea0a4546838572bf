#!/bin/bash
out=gpurun_out/r1w; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
bash tools/_ab.sh r1w base old
