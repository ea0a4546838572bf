#!/bin/bash
out=gpurun_out/r1av; mkdir -p $out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $out/tr1.json 2> $out/tr1.err; echo "rc=$?"
tail -3 $out/tr1.err; tail -c 600 $out/tr1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $out/tr1_ref.json 2> $out/tr1_ref.err; echo "rc=$?"
tail -c 400 $out/tr1_ref.json
