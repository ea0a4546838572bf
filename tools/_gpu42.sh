#!/bin/bash
out=gpurun_out/r1bi; mkdir -p $out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/b.json 2> $out/b.err; echo rc=$?
tail -2 $out/b.err
python -c "
import json
d=json.loads(open('$out/b.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['e2e']['value']), d['clocks'])"
