out=gpurun_out/r2g; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ingest.py tests/test_gpu_overlap.py tests/test_gpu_engine.py -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log; tail -2 $out/pytest.log
grep -E "^FAILED|^E  " $out/pytest.log | head -20
for cfg in block32 strip500; do
timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > $out/$cfg.json 2> $out/$cfg.err
python - $cfg $out/$cfg.json <<'PY'
import json, sys
j = json.loads(open(sys.argv[2]).read())
print(sys.argv[1], "value", round(j["value"]), "e2e", round(j["e2e"]["value"]), "e2e_ms", round(j["e2e"]["ms_per_step"],2),
      "pageable_ms", j["e2e_pageable"] and round(j["e2e_pageable"]["ms_per_step"],2), "files_ms", j["e2e_files"] and round(j["e2e_files"]["ms_per_step"],2))
PY
done
BMG_TIMELINE=1 timeout 300 python - > $out/timeline.log 2>&1 <<'PY'
import sys; sys.path.insert(0, ".")
import bench, torch
import paper_2505_22089_b200 as bm
from paper_2505_22089_b200.features import SyntheticScene, generate_synthetic
from paper_2505_22089_b200.engine import _feature_views
keep = []
def pin(n):
    t = torch.empty(n, dtype=torch.uint8, pin_memory=True); keep.append(t); return t.numpy()
imgs, _ = generate_synthetic(SyntheticScene(510, 8192, 10, 0.02, 0.2, 7), pinned=pin)
feats = {i - 10: fs for i, fs in enumerate(imgs) if i >= 10}
for i, fs in feats.items(): fs.image_id = i
plan = bm.read_plan("bench_data/plan_strip500.json")
hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
a = bm.DeviceArena(bm.arena_units_for(feats, plan.size_gpu), hf)
v = _feature_views(feats)
for _ in range(3): r = bm.execute_plan(plan, feats, a, views=v)
print("wall", r.metrics.wall_time_s, "device", r.metrics.device_ms)
PY
tail -60 $out/timeline.log > $out/timeline_tail.log
