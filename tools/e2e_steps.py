import sys, time
sys.path.insert(0, '.')
import torch, bench
import paper_2505_22089_b200 as bm
from paper_2505_22089_b200.engine import _feature_views
keep = []
def pinned(nbytes):
    t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True); keep.append(t); return t.numpy()
feats, plan = bench.build_workload("block32", 7, pinned)
hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
cap = bm.arena_units_for(feats, plan.size_gpu)
flat = bm.flatten_plan(plan); views = _feature_views(feats)
arena = bm.DeviceArena(cap, hf, 0)
ts = []
for i in range(20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = bm.execute_plan(plan, feats, arena, bm.ExecuteOptions(), flat=flat, views=views)
    ts.append((time.perf_counter() - t0) * 1e3)
print(" ".join(f"{t:.2f}" for t in ts))
