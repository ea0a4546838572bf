t=${1:-r1l}
mkdir -p gpurun_out/$t
timeout 900 python -m pytest tests/test_gpu_match.py tests/test_gpu_engine.py -q -x > gpurun_out/$t/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$t/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$t/bench.json 2> gpurun_out/$t/bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:match_ -s 2 -c 1 -o gpurun_out/$t/prof_match python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/$t/ncu.log 2>&1
tail -3 gpurun_out/$t/pytest_gpu.log; python -c "import json;d=json.load(open('gpurun_out/$t/bench.json'));print('value',d['value'],'e2e',d['e2e']['value'],d['kernel_ms_per_step'])"
