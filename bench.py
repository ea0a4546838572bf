#!/usr/bin/env python3
"""Benchmark: image match-pairs/sec at 8192 SIFT/img (BASELINE.json metric).

Workload (BASELINE config 2, "one MBR block"): 32 images x 8190 synthetic
SIFT-like descriptors (the reference generator, features.cpp:68-197, band 11;
the first 11 images of a 43-image scene are dropped so every image carries the
full 8190 descriptors), all 286 band pairs, scheduled by the reference's
iterate_schedule(16, 32) (bench_data/plan_block32.json: 2 block rows).  One
step = the whole execute_plan row loop (uploads, row means, codes, bucket
tables, cascade matching, result read-back) with verification off, exactly
the reference's `bandmatch match` path (bandmatch_cli.cpp:217-246).

  value  device time of the row loop on HBM-resident images (CUDA events on
         the compute stream), L2 flushed before every step
  e2e    wall time of the public execute_plan call from pinned host buffers:
         H2D of every image + rows + D2H of the matches, every step

Multi-GPU (torchrun): every rank runs its own block (seed 7 + rank) -- blocks
are independent units with no exchange step, so scaling is weak; times are
max over ranks.  `--impl reference` times the reference's CPU implementation
(oracle/_ref, the unmodified reference compiled in place) on rank 0 with every
host core.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "image match-pairs/sec at 8192 SIFT/img (1/2/4/8 B200) vs host-core CPU ref"
UNIT = "pairs/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
NCU_SUMMARY = ROOT / "profiles" / "ncu_summary.json"
FALLBACK_HBM = 6650.0

CONFIG_NO = {"pair1": 1, "block32": 2, "strip500": 3, "shard16k": 4}
CONFIGS = {
    # name: (generator n_images, ppi, band, dropped leading images, plan file)
    # BASELINE config 1: images (band, band+1) of an 11-band 8,192 scene
    "pair1": (13, 8192, 11, 11, "plan_pair1.json"),
    "block32": (43, 8192, 11, 11, "plan_block32.json"),
    "strip500": (510, 8192, 10, 10, "plan_strip500.json"),
    # BASELINE config 4 is 5,000 x 16,384 sharded over 2/4/8 GPUs: one
    # GPU's shard (640 images, band 15 = 30 neighbours); each rank its own
    "shard16k": (655, 16384, 15, 15, "plan_shard16k.json"),
}
# configs whose full reference run is minutes long: the CPU baseline is a
# timed sample (compute_codes of 32 images + match_pair of 128 pairs on all
# host threads) extrapolated to the plan's rows
SAMPLED = {"shard16k"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=list(CONFIGS), default="block32")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def build_workload(config: str, seed: int, pinned_alloc=None):
    """Scene + plan.  Returns ({id: FeatureSet}, plan, descriptors per image)."""
    import paper_2505_22089_b200 as bm
    from paper_2505_22089_b200.features import SyntheticScene, generate_synthetic

    n, ppi, band, drop, plan_file = CONFIGS[config]
    imgs, _ = generate_synthetic(SyntheticScene(n, ppi, band, 0.02, 0.2, seed), pinned=pinned_alloc)
    feats = {}
    for i, fs in enumerate(imgs[drop:]):
        fs.image_id = i
        feats[i] = fs
    plan = bm.read_plan(ROOT / "bench_data" / plan_file)
    return feats, plan


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    polled every 2 ms in a thread (nvidia-smi's 100 ms loop as fallback)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvml.h)
    NVML_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                 "hw_thermal_slowdown": 0x40}

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons) from NVML
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)

            def poll():
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                while not self.stop.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((float(sm), float(mx), {n for n, b in self.NVML_BITS.items() if bits & b}))
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=1)
            return
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for a, b, r in self.samples:
            sm.append(a)
            mx = max(mx, b)
            reasons |= r
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


def peaks():
    try:
        j = json.loads(PEAKS.read_text())
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def ncu_traffic(avg_ctas_per_launch):
    """DRAM bytes of one match launch from the committed `ncu --set full`
    capture, scaled by CTA count (one CTA = 1,024 queries of one pair) from
    the captured launch to this run's average launch (ncu: cold L2,
    serialised)."""
    try:
        m = json.loads(NCU_SUMMARY.read_text())["match_kernel"]
        g = m["metrics"]["launch__grid_size"]
        grid = float(str(g[0] if isinstance(g, (list, tuple)) else g).split()[0].replace(",", ""))
        return m["dram_bytes_per_launch"] / grid * avg_ctas_per_launch
    except Exception:
        return None


def reference_cpu(feats, plan_path, steps, warmup, threads):
    """oracle/_ref (the reference sources compiled in place) with rows'
    independent code computations and pair matches spread over `threads`."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Reference

    import paper_2505_22089_b200 as bm

    ref = Reference()
    imgs = {i: fs.descriptors for i, fs in feats.items()}
    hseed = bm.seed_for(42, "matching")
    times, pairs = [], 0
    for s in range(warmup + steps):
        done, m, wall = ref.execute_plan_threaded(plan_path, imgs, hseed, threads=threads)
        if s >= warmup:
            times.append(wall)
            pairs = done
    return pairs, times


def reference_cpu_sampled(feats, plan, threads):
    """Bounded CPU sample of the reference on `threads` threads, extrapolated
    to the plan: seconds = sum over rows of (needed images x t_codes + pairs x
    t_pair) / threads, with t_codes / t_pair measured per call on the sample."""
    import concurrent.futures as cf

    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Reference

    import paper_2505_22089_b200 as bm

    ref = Reference()
    hf = ref.make_hash_functions(bm.seed_for(42, "matching"))
    ids = sorted(feats)[:32]
    mean = np.mean(np.concatenate([feats[i].descriptors for i in ids]), axis=0).astype(np.float32)
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        codes = dict(zip(ids, ex.map(lambda i: ref.compute_codes(feats[i].descriptors, hf[0], hf[1], mean), ids)))
    t_codes = (time.perf_counter() - t0) * threads / len(ids)
    pairs = [(a, b) for a in ids for b in ids if a < b <= a + 15][:128]
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda p: ref.match_pair(feats[p[0]].descriptors, codes[p[0]], feats[p[1]].descriptors,
                                              codes[p[1]], (6, 8, 128)), pairs))
    t_pair = (time.perf_counter() - t0) * threads / len(pairs)
    secs, n_pairs = 0.0, 0
    for it in plan.iterations:
        for row in it.rows:
            needed = set(row.row_images)
            for b in row.blocks:
                needed.update(b.col_images)
                n_pairs += len(b.pairs)
                secs += len(b.pairs) * t_pair / threads
            secs += len(needed) * t_codes / threads
    sample = (f"extrapolated: compute_codes x {len(ids)} images ({t_codes:.2f} s each) + match_pair x "
              f"{len(pairs)} pairs ({t_pair:.3f} s each) on {threads} threads, scaled to the plan's "
              f"{n_pairs} pairs")
    return n_pairs, secs, sample


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_cfg, ppi, band, drop, plan_file = CONFIGS[args.config]
    plan_path = ROOT / "bench_data" / plan_file
    cores = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return 0
        feats, plan = build_workload(args.config, 7)
        sample = f"whole {args.config} plan per step"
        if args.config in SAMPLED:
            times = []
            for _ in range(args.steps):
                pairs, secs, sample = reference_cpu_sampled(feats, plan, cores)
                times.append(secs)
        else:
            pairs, times = reference_cpu(feats, plan_path, args.steps, args.warmup, cores)
            sample = f"whole {args.config} plan per step ({pairs} pairs)"
        mean_s = sum(times) / len(times)
        v = pairs / mean_s
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * mean_s,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (reference generator, features.cpp:68-197)",
                "impl": "reference",
                "config": {"workload": f"{args.config}: {len(feats)} images x {ppi - 2} desc, "
                                       f"{plan.pair_count()} pairs, plan {plan_file}",
                           "parallelism": f"{cores} host threads over each row's images/pairs"},
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    import torch.distributed as dist

    import paper_2505_22089_b200 as bm

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)

    pinned_keep = []

    def pinned_alloc(nbytes):
        t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        pinned_keep.append(t)
        return t.numpy()

    feats, plan = build_workload(args.config, 7 + rank, pinned_alloc)
    n_pairs = plan.pair_count()
    desc_bytes = sum(fs.descriptors.nbytes for fs in feats.values())
    avg_desc = desc_bytes / 512 / len(feats)
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    cap = bm.arena_units_for(feats, plan.size_gpu)
    flat = bm.flatten_plan(plan)
    from paper_2505_22089_b200.engine import _feature_views
    views = _feature_views(feats)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[dev])

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}")

    # ---- e2e: public API from pinned host memory, every byte every step ----
    arena_e2e = bm.DeviceArena(cap, hf, dev)
    opts = bm.ExecuteOptions()
    d2h = 0
    for _ in range(args.warmup):
        r = bm.execute_plan(plan, feats, arena_e2e, opts, flat=flat, views=views)
    barrier()
    e2e_times = []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = bm.execute_plan(plan, feats, arena_e2e, opts, flat=flat, views=views)
        e2e_times.append(time.perf_counter() - t0)
        d2h = 8 * (n_pairs + 1) + 8 * r.metrics.initial_matches
    barrier()
    e2e_step = max_over_ranks(sum(e2e_times) / len(e2e_times))
    e2e_matches = {(pm.query_image, pm.train_image): pm.matches for pm in r.matches}
    arena_e2e.matcher.close()

    # ---- value: the same row loop on HBM-resident images --------------------
    arena = bm.DeviceArena(cap * 2, hf, dev)
    for i, fs in feats.items():
        arena.upload(i, fs.descriptors)
    arena.matcher.synchronize()
    # reproject: the per-residency descriptor projections are recomputed in
    # every step, so the timed work is the complete row work
    vopts = bm.ExecuteOptions(retain=True, reproject=True)
    for _ in range(args.warmup):
        bm.execute_plan(plan, feats, arena, vopts, flat=flat, views=views)
    m = arena.matcher
    l0 = m.launch_count()
    dev_ms = []
    barrier()
    with ClockSampler(dev) as clocks:
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(2)  # L2 flush between timed steps (outside the event span)
            torch.cuda.synchronize()
            r = bm.execute_plan(plan, feats, arena, vopts, flat=flat, views=views)
            dev_ms.append(r.metrics.device_ms)
        barrier()
        t_wall = time.perf_counter() - t_wall0
    launches = m.launch_count() - l0
    got = {(pm.query_image, pm.train_image): pm.matches for pm in r.matches}
    consistent = got.keys() == e2e_matches.keys() and all(
        np.array_equal(got[k], e2e_matches[k]) for k in got)
    # kernel-timing pass (after the timed region): the same steps with the
    # rows on one stream, CUDA events around every launch on its stream.  In
    # the timed region consecutive rows overlap on two streams, so per-launch
    # event spans there would include the other row's kernels.
    sopts = bm.ExecuteOptions(retain=True, serial=True, reproject=True)
    m.set_profiling(True)
    for _ in range(args.steps):
        flush.fill_(3)
        torch.cuda.synchronize()
        bm.execute_plan(plan, feats, arena, sopts, flat=flat, views=views)
    match_ms, match_n = m.kernel_time("match")
    kt = {k: m.kernel_time(k) for k in ("project", "mean", "codes", "fixup", "tables", "match", "compact")}
    m.set_profiling(False)
    step_ms = max_over_ranks(sum(dev_ms) / len(dev_ms))
    value = world * n_pairs / (step_ms * 1e-3)
    e2e_value = world * n_pairs / e2e_step

    # roofline of the dominant kernel (the cascade match kernel):
    # algorithmic bytes per pair = both descriptor sets in f32 = 1024 * n
    pair_bytes = 0
    for it in plan.iterations:
        for row in it.rows:
            for b in row.blocks:
                for a, bb in b.pairs:
                    pair_bytes += feats[a].descriptors.nbytes + feats[bb].descriptors.nbytes
    per_launch_bytes = pair_bytes * args.steps / max(match_n, 1)
    avg_launch_s = match_ms * 1e-3 / max(match_n, 1)
    peak, peak_src = peaks()
    achieved = per_launch_bytes / avg_launch_s / 1e9 if avg_launch_s > 0 else 0.0
    step_ctas = sum(-(-len(feats[a].descriptors) // 1024)
                    for it in plan.iterations for row in it.rows for b in row.blocks for a, _ in b.pairs)
    traffic = ncu_traffic(step_ctas * args.steps / max(match_n, 1))

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic (reference generator features.cpp:68-197, seed 7+rank)",
            "config": {"workload": f"{args.config}: {len(feats)} images x {avg_desc:.0f} desc "
                                   f"(BASELINE config {CONFIG_NO[args.config]}), {n_pairs} pairs/GPU, "
                                   f"iterate_schedule plan {plan_file}",
                       "rows": sum(len(it.rows) for it in plan.iterations),
                       "k_nearest": 8, "ratio": 0.5, "hash": "L=6, m=8, n=128",
                       "l2": "flushed (512 MiB write) before every timed step",
                       "parallelism": f"row-block replicas, {world} GPU(s), no collective"},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": desc_bytes,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_step * 1e3,
                    "step_ms": [round(t * 1e3, 3) for t in e2e_times]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "match_kernel", "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": per_launch_bytes,
                         "avg_launch_ms": avg_launch_s * 1e3,
                         "timing": "CUDA events around each launch on its stream, serial-row pass "
                                   "of the same steps after the timed region"},
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items()},
            "results_consistent_e2e_vs_resident": consistent,
            "wall_s_timed": t_wall,
        }
    # CPU baseline: rank 0 at N=1 only, bounded sample of the same workload
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            if args.config in SAMPLED:
                pairs, secs, sample = reference_cpu_sampled(feats, plan, cores)
                line["cpu_baseline"] = {"value": pairs / secs, "unit": UNIT, "cores": cores,
                                        "kind": "reference", "sample": sample}
            else:
                pairs, times = reference_cpu(feats, plan_path, 1, 0, cores)
                line["cpu_baseline"] = {"value": pairs / times[0], "unit": UNIT, "cores": cores,
                                        "kind": "reference",
                                        "sample": f"whole {args.config} plan once ({pairs} pairs, "
                                                  f"{times[0]:.1f} s on {cores} threads)"}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": cores,
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.barrier(device_ids=[dev])
        dist.destroy_process_group()
    m.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
