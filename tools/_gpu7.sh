t=${1:-r1t}
mkdir -p gpurun_out/$t
timeout 900 python -m pytest tests/test_gpu_match.py tests/test_gpu_engine.py tests/test_gpu_binding.py -q -x > gpurun_out/$t/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$t/pytest_gpu.log
for v in 0 1; do BMG_MATCH_HALF=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$t/bench_$v.json 2> gpurun_out/$t/bench_$v.err; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:match -s 2 -c 1 -o gpurun_out/$t/prof_match python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/$t/ncu.log 2>&1
tail -1 gpurun_out/$t/pytest_gpu.log
for v in 0 1; do python -c "import json;d=json.load(open('gpurun_out/$t/bench_$v.json'));print('HALF=$v value',round(d['value']),'e2e',round(d['e2e']['value']))"; done
