out=gpurun_out/r2f; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log; tail -2 $out/pytest.log
grep -E "^FAILED" $out/pytest.log | head
for j in 0 1; do for cfg in block32 strip500; do
BMG_MATCH_JOIN=$j timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > $out/j${j}_$cfg.json 2> $out/j${j}_$cfg.err
python - $j $cfg $out/j${j}_$cfg.json <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[3]).read()); k = j["kernel_ms_per_step"]
    print(f"join={sys.argv[1]} {sys.argv[2]:9s} value {j['value']:9.0f} e2e {j['e2e']['value']:9.0f} match {k['match']:.3f} ms/step  ms/step {j['ms_per_step']:.3f} launches {j['gpu_launches']}")
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e)
PY
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_kernel -s 20 -c 1 -o $out/join python bench.py --config block32 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
