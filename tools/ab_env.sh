#!/bin/bash
# A/B of environment settings on the bench workloads (same libbmg):
# usage: gpurun -- bash tools/ab_env.sh TAG "ENV=.. ENV2=.." "..." ...   ("-" = no extra env)
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for rep in 1 2; do
i=0
for e in "$@"; do
  i=$((i+1))
  for cfg in block32 strip500; do
    f=$out/v${i}_${cfg}_$rep
    env $([ "$e" = "-" ] || echo $e) timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-files --no-retrieval > $f.json 2> $f.err
    python - "$e" "$cfg" "$f.json" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[3]).read()); k = j["kernel_ms_per_step"]
    print(f"{sys.argv[1][:40]:40s} {sys.argv[2]:9s} value {j['value']:9.0f} e2e {j['e2e']['value']:9.0f} ({j['e2e']['ms_per_step']:.2f} ms) page {j.get('e2e_pageable',{}).get('ms_per_step',0):.2f} ms  match {k['match']:.3f}")
except Exception as ex:
    print(sys.argv[1], sys.argv[2], "failed", ex)
PY
  done
done
done
