#!/bin/bash
# memcheck over the GPU suites (static cudart: compute-sanitizer intercepts the driver API)
out=gpurun_out/r1ai; mkdir -p $out
for t in test_gpu_match test_gpu_engine test_gpu_mean test_gpu_codes; do
  timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 77 --print-limit 20 \
    python -m pytest tests/$t.py -x -q > $out/memcheck_$t.log 2>&1; echo "$t rc=$?" >> $out/summary.txt
done
cat $out/summary.txt
for t in test_gpu_match test_gpu_engine; do grep -m3 "Invalid\|ERROR SUMMARY\|passed\|failed" $out/memcheck_$t.log; done
