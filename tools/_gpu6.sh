t=${1:-r1r}
mkdir -p gpurun_out/$t
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/$t/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$t/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$t/bench.json 2> gpurun_out/$t/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$t/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/$t/ncu_launch.log 2>&1
tail -1 gpurun_out/$t/pytest_gpu.log
python -c "import json;d=json.load(open('gpurun_out/$t/bench.json'));print('value',round(d['value']),'e2e',round(d['e2e']['value']), d['ms_per_step'])"
python tools/ncu_summary.py --round tmp --launches gpurun_out/$t/launches.csv | tail -22

