"""Generate the block-schedule inputs of the bench workloads with the
reference's own scheduler (iterate_schedule, mbr.cpp:321-376, via the test-only
oracle/_ref build).  The scheduler is out of scope for the GPU path (SURVEY
§2.1): its SchedulePlan is an *input*, so the plans are committed here as
fixtures under bench_data/.

  pair1     BASELINE config 1: the single pair (band, band+1) of an
            11-band scene, one 2-image row
  block32   BASELINE config 2: 32 images, band 11 (286 pairs),
            iterate_schedule(size_blk=16, size_gpu=32)
  strip500  BASELINE config 3: 500 images, band 10 (4945 pairs), CLI-default
            budget gpu_images=400 -> size_blk clamped to 200
            (bandmatch_cli.cpp:87-104)
  shard16k  BASELINE config 4, one GPU's shard: 640 of the 5,000 images at
            16,384 descriptors, band 15 (the 30 nearest neighbours), same
            CLI-default budget
  config4   BASELINE config 4 in full: 5,000 images at 16,384 descriptors,
            band 15 (74,880 pairs), same budget: 25 block rows
  strip1000 / strip2000 / strip4000
            the strip500 workload weak-scaled to 2 / 4 / 8 GPUs: a strip of
            500 N images, same band and budget (bench.py --gpus N shards it
            by rows, ~5,000 pairs per GPU)
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
from oracle_lib import Reference  # noqa: E402

OUT = ROOT / "bench_data"


def band_pairs(n, band):
    return np.array([(i, j) for i in range(n) for j in range(i + 1, min(n, i + band + 1))],
                    np.uint64)


def main():
    OUT.mkdir(exist_ok=True)
    r = Reference()
    for name, n, band, blk, gpu in [("pair1", 2, 1, 1, 2), ("block32", 32, 11, 16, 32), ("strip500", 500, 10, 200, 400),
                                    ("shard16k", 640, 15, 200, 400), ("config4", 5000, 15, 200, 400),
                                    ("strip1000", 1000, 10, 200, 400),
                                    ("strip2000", 2000, 10, 200, 400), ("strip4000", 4000, 10, 200, 400)]:
        r.iterate_schedule(np.arange(n), band_pairs(n, band), blk, gpu, OUT / f"plan_{name}.json")
        print(name, (OUT / f"plan_{name}.json").stat().st_size)


if __name__ == "__main__":
    main()
