"""Fraction of queries that take the matcher's exact top-K path on a
BASELINE-config row (diagnostics for the kLaneKeys choice).
usage: python tools/exact_probe.py [ppi] [n_imgs]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2505_22089_b200 as bm  # noqa: E402
from paper_2505_22089_b200.features import SyntheticScene, generate_synthetic  # noqa: E402

ppi = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
imgs, _ = generate_synthetic(SyntheticScene(n, ppi, min(11, n - 1), 0.02, 0.2, 7))
hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
with bm.Matcher(hf) as m:
    for i, f in enumerate(imgs):
        m.upload(i, np.ascontiguousarray(f.descriptors, np.float32))
    m.row(range(n))
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    m.match(pairs)
    m.synchronize()
    t = time.perf_counter()
    m.match(pairs)
    m.synchronize()
    dt = time.perf_counter() - t
    q = sum(len(imgs[i].descriptors) for i, _ in pairs)
    ex = m.exact_walk_count()
    print(f"ppi {ppi} imgs {n} pairs {len(pairs)} queries {q} exact {ex} ({ex / q:.5%}) "
          f"fp64 rerank {m.fixup_counts()[1]} match wall {dt * 1e3:.2f} ms")
