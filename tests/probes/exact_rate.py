"""Probe: how often K4's rare paths run on the bench workloads -- the exact
walk (a lane's key list may have dropped a needed key) and the FP64 re-rank
(the FP32 ratio certificate undecided). usage: python tests/probes/exact_rate.py [config]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import bench  # noqa: E402
import paper_2505_22089_b200 as bm  # noqa: E402
from paper_2505_22089_b200.features import SyntheticScene, generate_synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "block32"
n_cfg, ppi, band, drop, plan_file, _ = bench.resolve_config(cfg, 1, "weak")
plan = bm.read_plan(bench.ROOT / "bench_data" / plan_file)
imgs, _ = generate_synthetic(SyntheticScene(n_cfg, ppi, band, 0.02, 0.2, 7))
feats = {}
for i, fs in enumerate(imgs[drop:]):
    fs.image_id = i
    feats[i] = fs
hf = bm.make_hash_functions(bm.seed_for(bench.HASH_ROOT_SEED, "matching"))
out = []
with bm.Matcher(hf) as m:
    for fs in feats.values():
        m.upload(fs.image_id, fs.descriptors)
    for it in plan.iterations:
        for row in it.rows:
            need = sorted(set(row.row_images) | {i for blk in row.blocks for i in blk.col_images})
            pairs = [tuple(p) for blk in row.blocks for p in blk.pairs]
            m.row(need)
            m.match(pairs)
            e = m.exact_walk_count()
            bits, f = m.fixup_counts()
            q = sum(len(feats[a].descriptors) for a, _ in pairs)
            out.append({"pairs": len(pairs), "queries": q, "exact_walk": e, "exact_walk_frac": e / q,
                        "fp64_rerank": f, "fp64_rerank_frac": f / q, "fp64_code_bits": bits})
print(json.dumps({"config": cfg, "rows": out}))
