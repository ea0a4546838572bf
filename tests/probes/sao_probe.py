"""Timing probe (test infrastructure): host SAO filter (libbmg sao_filter,
knn_from_delaunay) vs the compiled reference's, on the matches of synthetic
scene pairs at 4k / 8k / 16k descriptors per image; results asserted equal.
usage: python tests/probes/sao_probe.py [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402

import paper_2505_22089_b200 as bm  # noqa: E402
from oracle_lib import Oracle, Reference  # noqa: E402
from paper_2505_22089_b200.verify import knn_from_delaunay, sao_filter  # noqa: E402
import test_sao  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ref, orc = Reference(), Oracle()
rows = []
for ppi in (4000, 8192, 16384):
    m, qk, tk = test_sao.scene_pair(ref, orc, ppi)
    pts = np.ascontiguousarray(qk[m[:, 0]][:, :2], np.float64)
    t_knn = t_sao = t_rknn = t_rsao = 1e9
    for _ in range(reps):
        t = time.perf_counter(); knn_from_delaunay(pts, 6); t_knn = min(t_knn, time.perf_counter() - t)
        t = time.perf_counter(); out = sao_filter(bm.PairMatches(1, 2, m), qk, tk); t_sao = min(t_sao, time.perf_counter() - t)
    for _ in range(max(1, reps // 3)):
        t = time.perf_counter(); ref.knn_from_delaunay(pts, 6); t_rknn = min(t_rknn, time.perf_counter() - t)
        t = time.perf_counter(); _, scores, _, _ = ref.sao_filter(m, qk, tk); t_rsao = min(t_rsao, time.perf_counter() - t)
    assert np.array_equal(out.scores, scores)
    r = {"ppi": ppi, "matches": int(len(m)), "knn_ms": t_knn * 1e3, "ref_knn_ms": t_rknn * 1e3,
         "sao_ms": t_sao * 1e3, "ref_sao_ms": t_rsao * 1e3, "speedup": t_rsao / t_sao}
    rows.append(r)
    print(json.dumps(r), flush=True)
