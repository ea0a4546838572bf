#!/bin/bash
# A/B of libbmg builds (tools/build_variant.sh) on the bench configs.
# usage: gpurun -- bash tools/ab_libs.sh <tag> <variant> [variant ...]   ("base" = libbmg.so)
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for cfg in block32 strip500; do
  for v in "$@"; do
    lib=paper_2505_22089_b200/libbmg.so; [ "$v" != base ] && lib=paper_2505_22089_b200/libbmg_$v.so
    BMG_LIBBMG=$PWD/$lib timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-files \
      > $out/${cfg}_$v.json 2> $out/${cfg}_$v.err
    python3 -c "
import json; d=json.loads(open('$out/${cfg}_$v.json').read().strip().splitlines()[-1])
print('$cfg', '$v', round(d['value']), round(d['e2e']['value']), round(d['kernel_ms_per_step']['match'],3), round(d['roofline']['frac'],4))" || tail -3 $out/${cfg}_$v.err
  done
done
