#!/bin/bash
out=gpurun_out/r1s; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_mean.py -x -q > $out/pytest_mean.log 2>&1; echo "rc=$?" >> $out/pytest_mean.log
BMG_TIMELINE=1 timeout 300 python tools/e2e_probe.py shard16k > $out/probe16k.log 2>&1
timeout 600 python bench.py --config shard16k --steps 5 --warmup 3 > $out/bench16k.json 2> $out/bench16k.err
tail -2 $out/pytest_mean.log; tail -30 $out/probe16k.log; cat $out/bench16k.json
