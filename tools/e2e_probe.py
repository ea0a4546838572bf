"""Where the end-to-end execute_plan time goes (bench workload, N=1): Python
wall, C++ wall (bmg_execute_plan), device span, per step.  BMG_TIMELINE=1
adds the per-row event timeline on stderr.
usage: python tools/e2e_probe.py [config] [steps] [pageable]"""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
import bench
import paper_2505_22089_b200 as bm
from paper_2505_22089_b200.engine import _feature_views
from paper_2505_22089_b200.features import SyntheticScene, generate_synthetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "strip500"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
pageable = len(sys.argv) > 3 and sys.argv[3] == "pageable"
keep = []
def pinned(nbytes):
    t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True); keep.append(t); return t.numpy()
n_cfg, ppi, band, drop, plan_file, _ = bench.resolve_config(cfg, 1, "weak")
plan = bm.read_plan(ROOT / "bench_data" / plan_file)
imgs, _ = generate_synthetic(SyntheticScene(n_cfg, ppi, band, 0.02, 0.2, 7), pinned=pinned)
feats = {}
for i, fs in enumerate(imgs[drop:]):
    fs.image_id = i
    feats[i] = fs
hf = bm.make_hash_functions(bm.seed_for(bench.HASH_ROOT_SEED, "matching"))
cap = bm.arena_units_for(feats, plan.size_gpu)
flat = bm.flatten_plan(plan)
if pageable:  # the reference's FeatureSet: pageable std::vector
    import numpy as np
    feats = {i: bm.FeatureSet(i, np.array(fs.descriptors)) for i, fs in feats.items()}
views = _feature_views(feats)
arena = bm.DeviceArena(cap, hf, 0)
opts = bm.ExecuteOptions()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
for i in range(steps):
    flush.fill_(1)
    torch.cuda.synchronize()
    print(f"---- step {i}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    r = bm.execute_plan(plan, feats, arena, opts, flat=flat, views=views)
    t1 = time.perf_counter()
    print(f"py {1e3*(t1-t0):7.3f} ms  c++ {1e3*r.metrics.wall_time_s:7.3f} ms  device {r.metrics.device_ms:7.3f} ms",
          flush=True)
    del r
