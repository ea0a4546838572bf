#!/bin/bash
# Validate the sharded bench on a one-GPU box: 2 ranks share the GPU (gloo).
tag=${1:-scale}; out=gpurun_out/$tag; mkdir -p $out
BMG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-files \
  > $out/bench_n2.json 2> $out/bench_n2.err; echo "rc=$?" >> $out/bench_n2.err
timeout 900 python bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $out/ref_n2.json 2> $out/ref_n2.err
tail -2 $out/bench_n2.err; cat $out/bench_n2.json | cut -c1-1500; cat $out/ref_n2.json | cut -c1-600
