out=gpurun_out/r2fin7; mkdir -p $out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 10 --warmup 3 > $out/ref.json 2> $out/ref.err; echo "ref rc=$?"
python - $out <<'PY'
import json, sys
o = sys.argv[1]
j = json.load(open(f"{o}/bench.json")); r = json.load(open(f"{o}/ref.json"))
print("ours", round(j["value"]), "e2e", round(j["e2e"]["value"]), "frac", round(j["roofline"]["frac"], 4), j["parity"]["status"], j["clocks"]["sm_mhz"], j["clocks"]["reasons"], "launches", j["gpu_launches"])
print("ref", round(r["value"], 1), r.get("impl"), r["config"]["workload"] == j["config"]["workload"])
PY
