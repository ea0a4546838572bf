#!/bin/bash
# BASELINE config 4 in full on one B200 (5,000 x 16,384, 74,880 pairs).
out=gpurun_out/${1:-c4}; mkdir -p $out
free -g > $out/free.txt
( while sleep 5; do free -g | sed -n 2p; nvidia-smi --query-gpu=memory.used --format=csv,noheader; done ) > $out/mem.log 2>&1 &
mon=$!
timeout 2400 python bench.py --config config4 --steps 3 --warmup 1 --no-files --no-retrieval \
  > $out/bench_config4.json 2> $out/bench_config4.err
echo "rc=$?" >> $out/bench_config4.err
kill $mon
tail -3 $out/bench_config4.err; cat $out/bench_config4.json | head -c 3000
