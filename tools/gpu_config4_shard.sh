#!/bin/bash
# BASELINE config 4 in full: one GPU, then the same plan sharded over 2 ranks
# that share the GPU (gloo barriers) -- the gathered result must equal the
# one-GPU result (result_digest).
out=gpurun_out/${1:-c4s}; mkdir -p $out
timeout 1800 python bench.py --config config4 --steps 2 --warmup 1 --no-files --no-retrieval --no-cpu-baseline \
  > $out/n1.json 2> $out/n1.err; echo "n1 rc=$?" >> $out/n1.err
BMG_BENCH_BACKEND=gloo timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config config4 --steps 2 --warmup 1 \
  --no-files --no-retrieval > $out/n2.json 2> $out/n2.err; echo "n2 rc=$?" >> $out/n2.err
python - $out <<'PY'
import json, sys
o = sys.argv[1]
a = json.loads(open(f"{o}/n1.json").read().strip().splitlines()[-1])
b = json.loads(open(f"{o}/n2.json").read().strip().splitlines()[-1])
print("N=1", a["value"], a["e2e"]["value"], a["result_digest"])
print("N=2 (one GPU, 2 ranks)", b["value"], b["e2e"]["value"], b["result_digest"], b["parity"]["digest_gpu"])
print("equal:", a["result_digest"]["digest"] == b["parity"]["digest_gpu"])
PY
