t=${1:-r1j}
mkdir -p gpurun_out/$t
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/$t/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$t/pytest_gpu.log
timeout 300 python tools/e2e_probe.py > gpurun_out/$t/probe.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$t/bench.json 2> gpurun_out/$t/bench.err
tail -15 gpurun_out/$t/pytest_gpu.log; cat gpurun_out/$t/probe.log | tail -4; cat gpurun_out/$t/bench.json; tail -3 gpurun_out/$t/bench.err
