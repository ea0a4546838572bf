t=${1:-r1v}
mkdir -p gpurun_out/$t
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/$t/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$t/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$t/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/$t/smoke.log
timeout 900 python bench.py --config strip500 --steps 3 --warmup 3 > gpurun_out/$t/bench_strip.json 2> gpurun_out/$t/bench_strip.err
timeout 1200 python tools/sweep.py --sizes 1024 2048 4096 8192 16384 32768 --out gpurun_out/$t/sweep.md > gpurun_out/$t/sweep.log 2>&1
tail -2 gpurun_out/$t/pytest_gpu.log; tail -2 gpurun_out/$t/smoke.log; cat gpurun_out/$t/bench_strip.json | cut -c1-600; tail -3 gpurun_out/$t/bench_strip.err; cat gpurun_out/$t/sweep.md
