#!/bin/bash
out=gpurun_out/r1ak; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_codes.py -x -q > $out/pytest_codes.log 2>&1; echo "rc=$?" >> $out/pytest_codes.log
BMG_PROJECT_SIMT=1 timeout 600 python -m pytest tests/test_gpu_codes.py -x -q > $out/pytest_codes_simt.log 2>&1; echo "rc=$?" >> $out/pytest_codes_simt.log
tail -12 $out/pytest_codes.log; tail -3 $out/pytest_codes_simt.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:project_tc -s 2 -c 1 -o $out/prof_project_tc python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/ncu_tc.log 2>&1; tail -2 $out/ncu_tc.log
