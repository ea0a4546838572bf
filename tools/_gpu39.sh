#!/bin/bash
out=gpurun_out/r1bb; mkdir -p $out
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 tests/cpp/_bin/test_reference_binding > $out/ms.log 2>&1; echo "rc=$?" >> $out/ms.log
head -40 $out/ms.log
