#!/bin/bash
# A/B of libbmg variants (tools/build_variant.sh) on the bench workloads:
# usage: gpurun -- bash tools/ab_variants.sh TAG VARIANT... ("default" = libbmg.so)
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for rep in 1 2; do
for v in "$@"; do
  lib=paper_2505_22089_b200/libbmg_$v.so; [ "$v" = default ] && lib=paper_2505_22089_b200/libbmg.so
  for cfg in block32 strip500; do
    BMG_LIBBMG=$PWD/$lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline \
      > $out/${v}_${cfg}_$rep.json 2> $out/${v}_${cfg}_$rep.err
    python - "$v" "$cfg" "$out/${v}_${cfg}_$rep.json" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[3]).read())
    k = j["kernel_ms_per_step"]
    print(f"{sys.argv[1]:10s} {sys.argv[2]:9s} value {j['value']:9.0f} e2e {j['e2e']['value']:9.0f} match {k['match']:.3f} ms/step  ms/step {j['ms_per_step']:.3f}")
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e)
PY
  done
done
done
