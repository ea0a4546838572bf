out=gpurun_out/r2k; mkdir -p $out
BMG_MATCH_ORDER=bucket timeout 900 python -m pytest tests/test_gpu_match.py tests/test_gpu_parity.py tests/test_gpu_engine.py -q -p no:cacheprovider -x > $out/pytest_bucket.log 2>&1; echo "rc=$?" >> $out/pytest_bucket.log; tail -2 $out/pytest_bucket.log
for rep in 1 2; do for o in index bucket; do for cfg in block32 strip500; do
BMG_MATCH_ORDER=$o timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-files > $out/${o}_$cfg.json 2> $out/${o}_$cfg.err
python - $o $cfg $out/${o}_$cfg.json <<'PY'
import json, sys
j = json.loads(open(sys.argv[3]).read()); k = j["kernel_ms_per_step"]
print(f"{sys.argv[1]:7s} {sys.argv[2]:9s} value {j['value']:9.0f} e2e {j['e2e']['value']:9.0f} match {k['match']:.3f} ms/step  ms/step {j['ms_per_step']:.3f}")
PY
done; done; done
