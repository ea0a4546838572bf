out=gpurun_out/r2i; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log; tail -2 $out/pytest.log
grep -E "^FAILED|^E  " $out/pytest.log | head -20
for cfg in block32 strip500; do
timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > $out/$cfg.json 2> $out/$cfg.err
python - $cfg $out/$cfg.json <<'PY'
import json, sys
j = json.loads(open(sys.argv[2]).read())
print(sys.argv[1], "value", round(j["value"]), "ms", round(j["ms_per_step"],3), "e2e", round(j["e2e"]["value"]), "e2e_ms", round(j["e2e"]["ms_per_step"],2),
      "pageable_ms", j["e2e_pageable"] and round(j["e2e_pageable"]["ms_per_step"],2), "files_ms", j["e2e_files"] and round(j["e2e_files"]["ms_per_step"],2))
print({k: round(v, 3) for k, v in j["kernel_ms_per_step"].items()})
PY
done
