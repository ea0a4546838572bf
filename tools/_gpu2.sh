mkdir -p gpurun_out/r1c
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 tests/cpp/_bin/test_reference_binding > gpurun_out/r1c/sanitizer.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r1c/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r1c/pytest_gpu.log
tail -30 gpurun_out/r1c/pytest_gpu.log; tail -30 gpurun_out/r1c/sanitizer.log
