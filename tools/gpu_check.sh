#!/bin/bash
# One GPU round trip: parity tests, smoke, bench (strip500 + block32).
# usage: gpurun --timeout 1800 -- bash tools/gpu_check.sh [tag] [pytest-args...]
tag=${1:-check}
shift
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider "$@" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
timeout 600 python bench.py --config block32 --steps 10 --warmup 3 > $out/bench_block32.json 2> $out/bench_block32.err
tail -3 $out/pytest_gpu.log; tail -1 $out/smoke.log; cat $out/bench.json
