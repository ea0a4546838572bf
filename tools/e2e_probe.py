"""Where the end-to-end execute_plan time goes (bench workload): Python wall,
C++ wall (bmg_execute_plan), device span, per step."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
import bench
import paper_2505_22089_b200 as bm
from paper_2505_22089_b200.engine import _feature_views

keep = []
def pinned(nbytes):
    t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True); keep.append(t); return t.numpy()
feats, plan = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "block32", 7, pinned)
hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
cap = bm.arena_units_for(feats, plan.size_gpu)
flat = bm.flatten_plan(plan)
views = _feature_views(feats)
arena = bm.DeviceArena(cap, hf, 0)
opts = bm.ExecuteOptions()
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = bm.execute_plan(plan, feats, arena, opts, flat=flat, views=views)
    t1 = time.perf_counter()
    print(f"py {1e3*(t1-t0):7.3f} ms  c++ {1e3*r.metrics.wall_time_s:7.3f} ms  device {r.metrics.device_ms:7.3f} ms")
