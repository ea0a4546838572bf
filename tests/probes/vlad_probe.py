"""Timing probe: bmg_encode_vlad on N synthetic 8,192-descriptor images
(pinned and pageable) vs the reference encode_vlad on the host cores.
usage: python tests/probes/vlad_probe.py [n_images] [cpu_images]"""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import paper_2505_22089_b200 as bm
from oracle_lib import Reference

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
ncpu = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ref = Reference()
imgs, _ = ref.generate_synthetic(12, 8192, 10, 0.02, 0.2, 7)
base = imgs[10:]
rng = np.random.default_rng(0)
allimgs = [base[i % 2][rng.permutation(len(base[i % 2]))] for i in range(n)]
cent, _ = ref.train_codebook(np.concatenate([b[::8] for b in base]), 64, 10, 3)
cb = bm.Codebook(64, cent)
m = bm.Matcher(bm.make_hash_functions(0))
pinned = [torch.from_numpy(a).pin_memory().numpy() for a in allimgs]
out = {}
for name, src in (("pinned", pinned), ("pageable", allimgs)):
    bm.encode_vlad_batch(src[:8], cb, m)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        got = bm.encode_vlad_batch(src, cb, m)
        ts.append(time.perf_counter() - t)
    out[name] = {"images_per_s": n / min(ts), "s": min(ts)}
L = bm.load()
import ctypes as C
L.bmg_set_profiling(m.handle, 1)
bm.encode_vlad_batch(pinned, cb, m)
tot, cnt = C.c_double(0), C.c_uint64(0)
L.bmg_kernel_time(m.handle, b"vlad", C.byref(tot), C.byref(cnt))
out["kernel_ms"] = tot.value
out["kernel_images_per_s"] = n / (tot.value / 1e3)
th = os.cpu_count()
t = time.perf_counter()
vals, degs = ref.encode_vlad_batch(allimgs[:ncpu], cent, threads=th)
dt = time.perf_counter() - t
out["cpu"] = {"images_per_s": ncpu / dt, "threads": th, "images": ncpu}
ok = all(np.array_equal(got[i].values.view(np.uint32), vals[i].view(np.uint32)) and got[i].degenerate == degs[i]
         for i in range(ncpu))
out["parity_first_cpu_images"] = ok
print(json.dumps(out))
