#!/usr/bin/env python3
"""Benchmark: image match-pairs/sec at 8192 SIFT/img (BASELINE.json metric).

Default workload (BASELINE config 3, "synthetic UAV strip", the largest
single-GPU 8,192-descriptor configuration): 500 images x 8,190 synthetic
SIFT-like descriptors from the reference generator (features.cpp:68-197, band
10: 20 neighbours per image; the 10 short leading images of a 510-image scene
are dropped), all 4,945 band pairs, scheduled by the reference's
iterate_schedule(200, 400) (bench_data/plan_strip500.json: 3 block rows).  One
step = the whole execute_plan row loop (uploads, row means, codes, bucket
tables, cascade matching, result read-back) with verification off, exactly
the reference's `bandmatch match` path (bandmatch_cli.cpp:217-246).
`--config block32` is BASELINE config 2 (one 32-image MBR block, 286 pairs;
verification off, like the reference arm), `pair1` config 1, `shard16k` one
GPU's shard of config 4.

  value  device time of the row loop on HBM-resident images (CUDA events on
         the compute streams), L2 flushed before every step
  e2e    wall time of the public execute_plan call from pinned host buffers:
         H2D of every image + rows + D2H of the matches, every step
         (e2e_pageable: the same from pageable buffers, like the reference's
         std::vector FeatureSet)
  parity the GPU match lists of the e2e run against the compiled reference
         (oracle/_ref) run on the same inputs in the cpu_baseline leg

Multi-GPU (torchrun, --gpus N): the plan is sharded (paper_2505_22089_b200.
multigpu): rows -- split by pairs where a row is larger than a rank's share --
are partitioned over the ranks with no collective on the data path; each rank
generates only the images its shard needs; matches are gathered to rank 0
through shared memory inside the timed region; times are max over ranks.
strip500 weak-scales by default (`--scaling weak`): N GPUs run the same UAV
strip with 500 N images (bench_data/plan_strip{500N}.json from the
reference's iterate_schedule, ~5,000 pairs per GPU); `--scaling strong`
shards the one 500-image plan.  `--impl reference` times the reference's CPU
implementation (oracle/_ref, the unmodified reference compiled in place) on
rank 0 with every host core, without loading this package.
"""
from __future__ import annotations

import argparse
import hashlib
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
HASH_ROOT_SEED = 42  # make_hash_functions(seed_for(42, "matching")), bandmatch_cli.cpp:225-226

CONFIG_NO = {"pair1": 1, "block32": 2, "strip500": 3, "shard16k": 4, "config4": 4}
CONFIGS = {
    # name: (generator n_images, ppi, band, dropped leading images, plan file)
    # BASELINE config 1: images (band, band+1) of an 11-band 8,192 scene
    "pair1": (13, 8192, 11, 11, "plan_pair1.json"),
    "block32": (43, 8192, 11, 11, "plan_block32.json"),
    "strip500": (510, 8192, 10, 10, "plan_strip500.json"),
    # BASELINE config 4 is 5,000 x 16,384 sharded over 2/4/8 GPUs: one
    # GPU's shard (640 images, band 15 = 30 neighbours)
    "shard16k": (655, 16384, 15, 15, "plan_shard16k.json"),
    # BASELINE config 4 in full (74,880 pairs, 25 block rows; ~42 GB of
    # descriptors: fits one B200's HBM, or shards over N GPUs)
    "config4": (5015, 16384, 15, 15, "plan_config4.json"),
}
# configs whose full reference run is minutes long: the CPU figure is a
# timed sample (compute_codes of 32 images + match_pair of 128 pairs on all
# host threads) extrapolated to the plan's rows
SAMPLED = {"shard16k", "config4"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=list(CONFIGS), default="strip500")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-files", action="store_true", help="skip the .feat-file e2e leg")
    p.add_argument("--no-retrieval", action="store_true", help="skip the VLAD encoding leg (f4)")
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                   help="N > 1 with strip500: weak = a strip of 500 N images (~5,000 pairs per GPU), "
                        "strong = the one 500-image plan sharded")
    return p.parse_args()


def resolve_config(config, world, scaling):
    """(generator n, ppi, band, drop, plan file, scaling label, images per GPU
    note).  strip500 at N > 1 weak-scales by default: the same UAV strip with
    500 N images (bench_data/plan_strip{500N}.json, the reference's
    iterate_schedule), so every GPU gets ~5,000 pairs of its own rows."""
    n_cfg, ppi, band, drop, plan_file = CONFIGS[config]
    if config == "strip500" and scaling == "weak":
        if world > 1:
            name = f"plan_strip{500 * world}.json"
            if (ROOT / "bench_data" / name).exists():
                return 500 * world + drop, ppi, band, drop, name, "weak"
            return n_cfg, ppi, band, drop, plan_file, "strong"
        return n_cfg, ppi, band, drop, plan_file, "weak"
    return n_cfg, ppi, band, drop, plan_file, "strong"


def plan_rows(plan_path):
    """[(pairs, needed image count)] per row in plan order, straight from the
    plan JSON (mbr.cpp:378-419 layout)."""
    j = json.loads(Path(plan_path).read_text())
    rows = []
    for it in j["iterations"]:
        for r in it["rows"]:
            need = set(r["row_images"])
            npairs = 0
            for blk in r["blocks"]:
                need.update(blk["col_images"])
                npairs += len(blk["pairs"])
            rows.append((npairs, len(need)))
    return rows


def workload_config(config, n_images, avg_desc, rows, resolved=None):
    """The `config` object, identical in both arms."""
    n_pairs = sum(p for p, _ in rows)
    n_cfg, ppi, band, drop, plan_file = (resolved or CONFIGS[config])[:5]
    if resolved and resolved[5] == "weak" and plan_file != CONFIGS[config][4]:
        config = f"{config} weak-scaled ({n_images} images)"
    return {"workload": f"{config}: BASELINE config {CONFIG_NO[config.split()[0]]}, {n_images} images x "
                        f"{avg_desc:.0f} desc, {n_pairs} pairs, {len(rows)} block rows, "
                        f"iterate_schedule plan {plan_file}, verification off",
            "rows": len(rows), "k_nearest": 8, "ratio": 0.5, "hash": "L=6, m=8, n=128",
            "scene": f"generate_synthetic(n={n_cfg}, ppi={ppi}, band={band}, sigma=0.02, "
                     f"outliers=0.2, seed=7), first {drop} images dropped",
            "l2": "GPU: flushed (512 MiB write) before every timed step"}


def digest(ids, offs, matches) -> str:
    """sha256 over the result in IdPair order: pair ids (u64), offsets (u64),
    (query_idx, train_idx) int32 pairs."""
    h = hashlib.sha256()
    for a, dt in ((ids, "<u8"), (offs, "<u8"), (matches, "<i4")):
        h.update(np.ascontiguousarray(a, dt).tobytes())
    return h.hexdigest()[:16]


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    polled every 2 ms in a thread (nvidia-smi's 100 ms loop as fallback, also
    when an NVML read fails mid-run).  The NVML handle is resolved from the
    CUDA device's PCI bus id, so CUDA_VISIBLE_DEVICES / torchrun remapping
    samples the right GPU."""

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
        self.t = None
        self.bus_id = None

    def _pci_bus_id(self):
        try:
            import torch
            p = torch.cuda.get_device_properties(self.device)
            return f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        except Exception:  # noqa: BLE001
            return None

    def _nvml_read(self, h):
        pynvml = self.nvml
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        try:
            bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except AttributeError:  # older bindings
            bits = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return float(sm), float(mx), {n for n, b in self.NVML_BITS.items() if bits & b}

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.bus_id = self._pci_bus_id()
            h = (pynvml.nvmlDeviceGetHandleByPciBusId(self.bus_id) if self.bus_id
                 else pynvml.nvmlDeviceGetHandleByIndex(self.device))
            self.samples.append(self._nvml_read(h))  # trial read: fail here, not in the thread

            def poll():
                while not self.stop.is_set():
                    try:
                        self.samples.append(self._nvml_read(h))
                    except Exception:  # noqa: BLE001
                        self._start_smi()
                        return
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001
            self._shutdown_nvml()
        self._start_smi()
        return self

    def _start_smi(self):
        if self.proc is not None:
            return
        try:
            target = self.bus_id or str(self.device)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", target, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def _shutdown_nvml(self):
        if self.nvml is not None:
            try:
                self.nvml.nvmlShutdown()
            except Exception:  # noqa: BLE001
                pass
        self.nvml = None

    def __exit__(self, *a):
        self.stop.set()
        if self.t is not None:
            self.t.join(timeout=1)
        self._shutdown_nvml()
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
        src = "+".join(s for s, on in (("nvml", self.samples), ("nvidia-smi", self.lines)) if on)
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": src}


def peaks():
    try:
        j = json.loads(PEAKS.read_text())
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def sm_max_mhz():
    try:
        return float(json.loads(PEAKS.read_text())["sm_max_mhz"])
    except Exception:  # noqa: BLE001
        return 1965.0  # B200 boost clock (B200_PROFILING.md)


# queries per match CTA (csrc/bmg_internal.h BMG_MATCH_QUERIES): scales the
# committed ncu capture's per-CTA figures to this run's launches
MATCH_QUERIES_PER_CTA = 2048


def ncu_traffic(avg_ctas_per_launch):
    """DRAM bytes of one match launch from the committed `ncu --set full`
    capture, scaled by CTA count (one CTA = 2,048 queries of one pair) from
    the captured launch to this run's average launch (ncu: cold L2,
    serialised)."""
    try:
        m = json.loads(NCU_SUMMARY.read_text())["match_kernel"]
        g = m["metrics"]["launch__grid_size"]
        grid = float(str(g[0] if isinstance(g, (list, tuple)) else g).split()[0].replace(",", ""))
        return m["dram_bytes_per_launch"] / grid * avg_ctas_per_launch
    except Exception:  # noqa: BLE001
        return None


def ncu_inst_per_cta():
    """Warp instructions per match CTA (1,024 queries of one pair) from the
    committed `ncu --set full` capture: the issue-slot roofline's work."""
    try:
        m = json.loads(NCU_SUMMARY.read_text())["match_kernel"]["metrics"]
        num = lambda v: float(str(v[0] if isinstance(v, (list, tuple)) else v).split()[0].replace(",", ""))
        return num(m["smsp__inst_executed.sum"]) / num(m["launch__grid_size"])
    except Exception:  # noqa: BLE001
        return None


MICROBENCH = ROOT / "profiles" / "r2_microbench.json"


def microbench_peaks() -> dict:
    try:
        return json.loads(MICROBENCH.read_text())
    except Exception:  # noqa: BLE001
        return {}


def candidates_per_query(m, plan, feats, samples=16):
    """Duplicate-inclusive candidates per query (the union walk's entries
    before dedup, hashmatch.cpp:154-167) on up to `samples` pairs of the
    plan's largest row, from the GPU's own codes of that row."""
    rows = [r for it in plan.iterations for r in it.rows]
    if not rows:
        return 0.0
    row = max(rows, key=lambda r: sum(len(b.pairs) for b in r.blocks))
    pairs = [p for b in row.blocks for p in b.pairs][:samples]
    if not pairs:
        return 0.0
    m.row(row.needed())
    nb = 1 << m.hf.params.coarse_bits
    codes = {}
    for i in {x for p in pairs for x in p}:
        codes[i] = m.codes(i, len(feats[i].descriptors)).coarse
    cand = q = 0
    for a, b in pairs:
        for t in range(codes[a].shape[1]):
            ca = np.bincount(codes[a][:, t], minlength=nb)
            cb = np.bincount(codes[b][:, t], minlength=nb)
            cand += int((ca.astype(np.int64) * cb).sum())
        q += codes[a].shape[0]
    return cand / q


# ---------------------------------------------------------------------------
# the reference (CPU) legs: oracle/_ref only
# ---------------------------------------------------------------------------
def _reference():
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Reference
    return Reference()


def reference_sampled(ref, images, rows, threads):
    """Bounded CPU sample of the reference on `threads` threads, extrapolated
    to the plan: seconds = sum over rows of (needed images x t_codes + pairs x
    t_pair) / threads, with t_codes / t_pair measured per call on the sample.
    images: {id: (n,128) f32} (at least the first 32 ids)."""
    import concurrent.futures as cf

    hf = ref.make_hash_functions(ref.seed_for(HASH_ROOT_SEED, "matching"))
    ids = sorted(images)[:32]
    mean = np.mean(np.concatenate([images[i] for i in ids]), axis=0).astype(np.float32)
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        codes = dict(zip(ids, ex.map(lambda i: ref.compute_codes(images[i], hf[0], hf[1], mean), ids)))
    t_codes = (time.perf_counter() - t0) * threads / len(ids)
    pairs = [(a, b) for a in ids for b in ids if a < b <= a + 15][:128]
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda p: ref.match_pair(images[p[0]], codes[p[0]], images[p[1]], codes[p[1]],
                                              (6, 8, 128)), pairs))
    t_pair = (time.perf_counter() - t0) * threads / len(pairs)
    secs = sum(p * t_pair + n * t_codes for p, n in rows) / threads
    n_pairs = sum(p for p, _ in rows)
    sample = (f"extrapolated: compute_codes x {len(ids)} images ({t_codes:.2f} s each) + match_pair x "
              f"{len(pairs)} pairs ({t_pair:.3f} s each) on {threads} threads, scaled to the plan's "
              f"{n_pairs} pairs")
    return n_pairs, secs, sample


def reference_arm(args):
    """`--impl reference`: the reference's own CPU code on every host core.
    Inputs come from the reference generator (oracle/_ref) -- this package is
    not imported.  Step s runs block row s mod rows of the plan in full (its
    mean, compute_codes of its needed images, match_pair of its pairs: the
    row body of engine.cpp:433-489) so the run stays within minutes; value =
    pairs / seconds over the timed steps."""
    resolved = resolve_config(args.config, args.gpus, args.scaling)
    n_cfg, ppi, band, drop, plan_file, scaling = resolved
    plan_path = ROOT / "bench_data" / plan_file
    rows = plan_rows(plan_path)
    cores = os.cpu_count() or 1
    ref = _reference()
    hseed = ref.seed_for(HASH_ROOT_SEED, "matching")
    if args.config in SAMPLED:
        images, _ = ref.generate_synthetic(n_cfg, ppi, band, 0.02, 0.2, 7)
        images = {i - drop: d for i, d in enumerate(images) if i >= drop}
        n_images = len(images)
        avg = sum(len(d) for d in images.values()) / n_images
        tot_s, tot_p = 0.0, 0
        for _ in range(args.steps):
            p, s, sample = reference_sampled(ref, images, rows, cores)
            tot_s += s
            tot_p += p
        warm = "none (extrapolated sample)"
    else:
        table = ref.synth_features(n_cfg, ppi, band, 0.02, 0.2, 7, drop)
        n_images = table.n
        avg = sum(table.count(i) for i in range(n_images)) / n_images
        ref.execute_plan_rows(plan_path, table, hseed, threads=cores, row_begin=0, row_end=1)
        warm = "one block row (a CPU has no JIT or cache state to warm beyond that)"
        tot_s, tot_p = 0.0, 0
        for s in range(args.steps):
            r = s % len(rows)
            p, _, wall, _ = ref.execute_plan_rows(plan_path, table, hseed, threads=cores,
                                                  row_begin=r, row_end=r + 1)
            tot_s += wall
            tot_p += p
        sample = (f"{args.steps} steps, step s = block row s mod {len(rows)} of the plan in full "
                  f"(row mean + compute_codes of its needed images + match_pair of its pairs)")
        table.free()
    v = tot_p / tot_s
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator features.cpp:68-197, oracle/_ref)",
            "impl": "reference",
            "config": workload_config(args.config, n_images, avg, rows, resolved),
            "parallelism": f"{cores} host threads over each row's images / pairs",
            "cpu_warmup": warm,
            "host_cpu": cpu_model(),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def sampled_parity(ref, hseed, images, plan_path, gpu_flat, cores, n_pairs=48):
    """Parity on a sample of a long plan: the reference runs the LAST block
    row with its whole needed set (so its mean and codes are the full row's)
    but only the first `n_pairs` pairs of its blocks; their match lists are
    compared with the GPU's for the same pairs."""
    import tempfile

    j = json.loads(Path(plan_path).read_text())
    it = j["iterations"][-1]
    row = json.loads(json.dumps(it["rows"][-1]))
    left = n_pairs
    for blk in row["blocks"]:
        blk["pairs"] = blk["pairs"][:left]
        left -= len(blk["pairs"])
    row["evict_after"] = []
    sub = dict(j)
    sub["iterations"] = [dict(it, rows=[row])]
    need = set(row["row_images"])
    for blk in row["blocks"]:
        need.update(blk["col_images"])
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(sub, f)
    try:
        done, _, wall, res = ref.execute_plan_rows(f.name, {i: images[i] for i in sorted(need)}, hseed,
                                                   threads=cores, want_matches=True)
    finally:
        os.unlink(f.name)
    ri, ro, rm = res
    gi, go, gm = gpu_flat
    where = {(int(a), int(b)): p for p, (a, b) in enumerate(gi)}
    eq = True
    mine = []
    for p, (a, b) in enumerate(ri):
        g = where.get((int(a), int(b)))
        got = gm[go[g]:go[g + 1]] if g is not None else None
        if got is None or not np.array_equal(got, rm[ro[p]:ro[p + 1]]):
            eq = False
        mine.append(got if got is not None else np.zeros((0, 2), np.int32))
    go_s = np.concatenate([[0], np.cumsum([len(x) for x in mine])]).astype(np.uint64)
    gm_s = np.concatenate(mine) if mine else np.zeros((0, 2), np.int32)
    return {"status": "equal" if eq else "DIFFERENT", "pairs": int(len(ri)), "matches": int(len(rm)),
            "digest_gpu": digest(ri, go_s, gm_s), "digest_reference": digest(ri, ro, rm),
            "reference": (f"oracle/_ref row body on a sample: the plan's last block row with its whole "
                          f"needed set ({len(need)} images: the full row mean and codes), its first "
                          f"{len(ri)} pairs; {wall:.1f} s on {cores} threads")}


def parity_leg(feats, plan_path, rows, config, gpu_flat, cores):
    """Runs the compiled reference on the repo arm's own inputs (same
    arrays): its CPU time is the line's cpu_baseline, its match lists are
    compared with the GPU's (the e2e run's result)."""
    ref = _reference()
    hseed = ref.seed_for(HASH_ROOT_SEED, "matching")
    images = {i: fs.descriptors for i, fs in feats.items()}
    if config in SAMPLED:
        p, secs, sample = reference_sampled(ref, images, rows, cores)
        cpu = {"value": p / secs, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample}
        return cpu, sampled_parity(ref, hseed, images, plan_path, gpu_flat, cores)
    table = ref.feature_table(images)
    done, m, wall, res = ref.execute_plan_rows(plan_path, table, hseed, threads=cores, want_matches=True)
    table.free()
    cpu = {"value": done / wall, "unit": UNIT, "cores": cores, "kind": "reference",
           "sample": f"whole {config} plan once ({done} pairs, {wall:.1f} s on {cores} threads)"}
    gi, go, gm = gpu_flat
    ri, ro, rm = res
    eq = (np.array_equal(gi, ri) and np.array_equal(go, ro) and np.array_equal(gm, rm))
    par = {"status": "equal" if eq else "DIFFERENT", "pairs": int(len(ri)), "matches": int(len(rm)),
           "digest_gpu": digest(gi, go, gm), "digest_reference": digest(ri, ro, rm),
           "reference": "oracle/_ref execute_plan row body (compute_codes + match_pair), same inputs"}
    if not eq:
        par["pairs_differing"] = int(sum(
            1 for p in range(min(len(gi), len(ri)))
            if not np.array_equal(gm[go[p]:go[p + 1]], rm[ro[p]:ro[p + 1]])))
    return cpu, par


def retrieval_leg(bm, m, feats, cores, cpu=True, cpu_images=32):
    """encode_vlad (retrieval.cpp:160-205) of every bench
    image on the B200 (bmg_encode_vlad, pageable FeatureSets as select_pairs
    passes them, and pinned) against the compiled reference's encode_vlad on
    the host cores over a sample, with bit-exact parity on the sample.  The
    codebook is 64 descriptors sampled from the images (train_codebook's
    initial centroids; retrieval.cpp:66-96)."""
    import ctypes as C
    imgs = [feats[i].descriptors for i in sorted(feats)]
    rng = np.random.default_rng(64)
    pool = np.concatenate([im[rng.integers(0, len(im), 4)] for im in imgs])
    cent = np.ascontiguousarray(pool[rng.choice(len(pool), 64, replace=False)], np.float32)
    cb = bm.Codebook(64, cent)
    L = bm.load()
    pageable = [np.array(a) for a in imgs]  # the bench images live in pinned memory

    def best(src, reps=2):
        bm.encode_vlad_batch(src[:4], cb, m)
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            r = bm.encode_vlad_batch(src, cb, m)
            ts.append(time.perf_counter() - t)
        return min(ts), r

    e2e_pageable, got = best(pageable)
    e2e_pinned, _ = best(imgs)
    L.bmg_set_profiling(m.handle, 1)  # (clears earlier timers)
    bm.encode_vlad_batch(imgs, cb, m)
    tot, cnt = C.c_double(0), C.c_uint64(0)
    L.bmg_kernel_time(m.handle, b"vlad", C.byref(tot), C.byref(cnt))
    L.bmg_set_profiling(m.handle, 0)
    del pageable
    n = len(imgs)
    out = {"workload": f"encode_vlad of the {n} bench images (k_words 64)", "unit": "images/s",
           "e2e_pageable": n / e2e_pageable, "e2e_pinned": n / e2e_pinned,
           "kernels": n / (tot.value / 1e3) if tot.value > 0 else None,
           "h2d_bytes": int(sum(a.nbytes for a in imgs))}
    if cpu:
        ref = _reference()
        k = min(cpu_images, n)
        t = time.perf_counter()
        vals, degs = ref.encode_vlad_batch(imgs[:k], cent, threads=cores)
        dt = time.perf_counter() - t
        eq = all(np.array_equal(got[i].values.view(np.uint32), vals[i].view(np.uint32))
                 and got[i].degenerate == degs[i] for i in range(k))
        out["cpu_baseline"] = {"value": k / dt, "unit": "images/s", "cores": cores, "kind": "reference",
                               "sample": f"first {k} images"}
        out["parity"] = "equal" if eq else "DIFFERENT"
    # train_codebook (retrieval.cpp:56-158) on a training pool drawn from the
    # images (every 100th descriptor), k_words 64, up to 10 Lloyd iterations:
    # the device against the reference's single-threaded loops
    pool_tc = np.ascontiguousarray(np.concatenate([im[::100] for im in imgs]), np.float32)
    bm.train_codebook(pool_tc[:4096], 64, 2, 3, matcher=m)  # warm
    t = time.perf_counter()
    hist = []
    cb_gpu = bm.train_codebook(pool_tc, 64, 10, 3, sse_history=hist, matcher=m)
    t_gpu = time.perf_counter() - t
    tc = {"pool": int(len(pool_tc)), "k_words": 64, "max_iters": 10, "iterations": len(hist),
          "gpu_ms": t_gpu * 1e3}
    if cpu:
        t = time.perf_counter()
        cent_ref, sse_ref = _reference().train_codebook(pool_tc, 64, 10, 3)
        tc["reference_ms"] = (time.perf_counter() - t) * 1e3
        tc["reference_threads"] = 1
        tc["parity"] = ("equal" if np.array_equal(np.asarray(cb_gpu.centroids, np.float32).view(np.uint32),
                                                  cent_ref.view(np.uint32))
                        and np.array_equal(np.asarray(hist), sse_ref) else "DIFFERENT")
    out["train_codebook"] = tc
    return out


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args) if rank == 0 else 0

    import torch
    import torch.distributed as dist

    import paper_2505_22089_b200 as bm
    from paper_2505_22089_b200 import multigpu
    from paper_2505_22089_b200.engine import _feature_views
    from paper_2505_22089_b200.features import SyntheticScene, generate_synthetic, synthetic_counts

    resolved = resolve_config(args.config, world, args.scaling)
    n_cfg, ppi, band, drop, plan_file, scaling = resolved
    plan_path = ROOT / "bench_data" / plan_file
    rows = plan_rows(plan_path)
    cores = os.cpu_count() or 1
    # BMG_BENCH_BACKEND=gloo: ranks may share a GPU (validation of the
    # sharded path on a one-GPU box); the driver's runs use NCCL, one GPU each
    backend = os.environ.get("BMG_BENCH_BACKEND", "nccl")
    dev = local % max(torch.cuda.device_count(), 1) if world > 1 else 0
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group(backend)

    plan = bm.read_plan(plan_path)
    n_pairs = plan.pair_count()
    # this rank's shard of the one plan (the whole plan at N=1)
    sub = multigpu.shard_plan(plan, world)[rank] if world > 1 else plan
    mine = multigpu.needed_images(sub)

    pinned_keep = []

    def pinned_alloc(nbytes):
        t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        pinned_keep.append(t)
        return t.numpy()

    # the scene, generated into pinned memory: only the images this rank needs
    keep = {i + drop for i in mine}
    imgs, _ = generate_synthetic(SyntheticScene(n_cfg, ppi, band, 0.02, 0.2, 7), pinned=pinned_alloc,
                                 keep=keep)
    feats = {}
    for i, fs in enumerate(imgs[drop:]):
        if fs is not None:
            fs.image_id = i
            feats[i] = fs
    counts_all = synthetic_counts(SyntheticScene(n_cfg, ppi, band, 0.02, 0.2, 7))[drop:]
    n_images = len(counts_all)
    avg_desc = float(counts_all.sum()) / n_images
    my_pairs = sub.pair_count()
    desc_bytes = sum(fs.descriptors.nbytes for fs in feats.values())
    hf = bm.make_hash_functions(bm.seed_for(HASH_ROOT_SEED, "matching"))
    cap = bm.arena_units_for(feats, plan.size_gpu) if feats else 1
    flat = bm.flatten_plan(sub)
    views = _feature_views(feats)

    def dist_barrier():
        if backend == "nccl":
            dist.barrier(device_ids=[dev])
        else:
            dist.barrier()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist_barrier()

    def reduce_over_ranks(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x: float) -> float:
        return reduce_over_ranks(x, dist.ReduceOp.MAX) if world > 1 else x

    def sum_over_ranks(x: float) -> float:
        return reduce_over_ranks(x, dist.ReduceOp.SUM) if world > 1 else x

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}")

    # ---- e2e: the public API from pinned host memory, every byte every step;
    # at N>1 the shared-memory gather of every rank's matches to rank 0 is
    # inside the timed region
    arena_e2e = bm.DeviceArena(cap, hf, dev)
    opts = bm.ExecuteOptions()

    def e2e_step(step):
        r = bm.execute_plan(sub, feats, arena_e2e, opts, flat=flat, views=views)
        if world > 1:
            got = multigpu.gather_results(r, rank, world, dist_barrier,
                                          f"{os.environ.get('MASTER_PORT', '0')}_{step}")
            return r, got
        return r, None

    # the previous step's result is released before the next call, so the
    # result's pinned log comes back from the process-wide pool every step
    r = got = None
    for w in range(args.warmup):
        r = got = None
        r, got = e2e_step(f"w{w}")
    barrier()
    e2e_times, d2h = [], 0
    for s in range(args.steps):
        flush.fill_(1)
        r = got = None
        barrier()
        t0 = time.perf_counter()
        r, got = e2e_step(s)
        e2e_times.append(time.perf_counter() - t0)
        d2h = 8 * (my_pairs + 1) + 8 * r.metrics.initial_matches
    barrier()
    e2e_step_s = max_over_ranks(sum(e2e_times) / len(e2e_times))
    h2d_all = sum_over_ranks(desc_bytes)
    d2h_all = sum_over_ranks(d2h)
    gpu_flat = multigpu.result_flat(r) if world == 1 else (got[0].flat() if rank == 0 else None)
    e2e_result = r
    arena_e2e.matcher.close()

    # ---- e2e from pageable host memory (the reference's FeatureSet is a
    # std::vector): the same call, H2D through the staging ring
    page_ms = None
    if world == 1:
        pfeats = {i: bm.FeatureSet(i, np.array(fs.descriptors)) for i, fs in feats.items()}
        pviews = _feature_views(pfeats)
        arena_p = bm.DeviceArena(cap, hf, dev)
        bm.execute_plan(sub, pfeats, arena_p, opts, flat=flat, views=pviews)
        pt = []
        for _ in range(min(args.steps, 5)):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bm.execute_plan(sub, pfeats, arena_p, opts, flat=flat, views=pviews)
            pt.append(time.perf_counter() - t0)
        page_ms = 1e3 * sum(pt) / len(pt)
        arena_p.matcher.close()
        del pfeats, pviews
    # ---- e2e from .feat files (streamed as images upload, f2): files written
    # first (outside the timing) to a temp dir; page cache warm
    files_ms = None
    if world == 1 and not args.no_files:
        import shutil
        import tempfile

        from paper_2505_22089_b200.features import write_features
        tmpd = Path(tempfile.mkdtemp(prefix="bmg_feat_"))
        try:
            fpaths = {}
            for i, fs in feats.items():
                fpaths[i] = str(tmpd / f"{i:06d}.feat")
                write_features(fpaths[i], bm.FeatureSet(i, fs.descriptors))
            fviews = _feature_views(fpaths)
            arena_f = bm.DeviceArena(cap, hf, dev)
            bm.execute_plan(sub, fpaths, arena_f, opts, flat=flat, views=fviews)
            ft = []
            for _ in range(min(args.steps, 3)):
                flush.fill_(1)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                bm.execute_plan(sub, fpaths, arena_f, opts, flat=flat, views=fviews)
                ft.append(time.perf_counter() - t0)
            files_ms = 1e3 * sum(ft) / len(ft)
            arena_f.matcher.close()
        finally:
            shutil.rmtree(tmpd, ignore_errors=True)

    # ---- value: the same row loop on HBM-resident images ---------------------
    # every image of the rank stays resident (config 4: ~42 GB of
    # descriptors + projections; fits one B200)
    arena = bm.DeviceArena(max(cap * 2, sum(len(fs.descriptors) for fs in feats.values()) + 1), hf, dev)
    for i, fs in feats.items():
        arena.upload(i, fs.descriptors)
    arena.matcher.synchronize()
    # reproject: the per-residency descriptor projections are recomputed in
    # every step, so the timed work is the complete row work
    vopts = bm.ExecuteOptions(retain=True, reproject=True)
    for _ in range(args.warmup):
        bm.execute_plan(sub, feats, arena, vopts, flat=flat, views=views)
    m = arena.matcher
    l0 = m.launch_count()
    dev_ms = []
    barrier()
    # NVTX range "value": lets ncu capture the timed loop's launches alone
    # (tools/gpu_prof.sh: --nvtx --nvtx-include value/)
    with ClockSampler(dev) as clocks:
        torch.cuda.nvtx.range_push("value")
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(2)  # L2 flush between timed steps (outside the event span)
            barrier()
            rv = bm.execute_plan(sub, feats, arena, vopts, flat=flat, views=views)
            dev_ms.append(rv.metrics.device_ms)
        barrier()
        t_wall = time.perf_counter() - t_wall0
        torch.cuda.nvtx.range_pop()
    launches = m.launch_count() - l0
    vi, vo, vm = multigpu.result_flat(rv)
    ei, eo, em = multigpu.result_flat(e2e_result)
    consistent = (np.array_equal(vi, ei) and np.array_equal(vo, eo) and np.array_equal(vm, em))
    # kernel-timing pass (after the timed region): the same steps with the
    # rows on one stream, CUDA events around every launch on its stream.  In
    # the timed region consecutive rows overlap on two streams, so per-launch
    # event spans there would include the other row's kernels.
    sopts = bm.ExecuteOptions(retain=True, serial=True, reproject=True)
    m.set_profiling(True)
    for _ in range(args.steps):
        flush.fill_(3)
        torch.cuda.synchronize()
        bm.execute_plan(sub, feats, arena, sopts, flat=flat, views=views)
    match_ms, match_n = m.kernel_time("match")
    kt = {k: m.kernel_time(k) for k in ("project", "mean", "codes", "fixup", "tables", "match", "compact")}
    m.set_profiling(False)
    step_ms = max_over_ranks(sum(dev_ms) / len(dev_ms))
    value = n_pairs / (step_ms * 1e-3)
    e2e_value = n_pairs / e2e_step_s

    # roofline of the dominant kernel (the cascade match kernel):
    # algorithmic bytes per pair = both descriptor sets in f32 = 1024 * n
    pair_bytes = 0
    step_ctas = 0
    for it in sub.iterations:
        for row in it.rows:
            for blk in row.blocks:
                for a_, b_ in blk.pairs:
                    pair_bytes += feats[a_].descriptors.nbytes + feats[b_].descriptors.nbytes
                    step_ctas += -(-len(feats[a_].descriptors) // MATCH_QUERIES_PER_CTA)
    per_launch_bytes = pair_bytes * args.steps / max(match_n, 1)
    avg_launch_s = match_ms * 1e-3 / max(match_n, 1)
    peak, peak_src = peaks()
    achieved = per_launch_bytes / avg_launch_s / 1e9 if avg_launch_s > 0 else 0.0
    traffic = ncu_traffic(step_ctas * args.steps / max(match_n, 1))
    consistent_all = max_over_ranks(0.0 if consistent else 1.0) == 0.0
    # secondary rooflines of the match kernel: POPC and the
    # candidate-code gathers, from the duplicate-inclusive candidates per
    # query measured on a sample of the largest row's pairs (bucket sizes of
    # the GPU's own codes: sum over tables and buckets of |Q_b| * |T_b|)
    cand_q = candidates_per_query(m, sub, feats)
    micro = microbench_peaks()
    queries_per_launch = sum(len(feats[a_].descriptors) for it in sub.iterations for row in it.rows
                             for blk in row.blocks for a_, _ in blk.pairs) * args.steps / max(match_n, 1)
    fw = 2  # u64 words per fine code (128 bits)
    popc_per_launch = queries_per_launch * cand_q * 2 * fw
    gather_per_launch = queries_per_launch * cand_q * (8 * fw + 4)

    def issue_roofline():
        # the binding resource of K4 (ncu: issue-bound, ALU pipe ~64%): warp
        # instructions per launch (committed ncu capture, per CTA x this
        # run's CTAs per launch) / launch time, against 4 issue slots per SM
        # per cycle at the sampled SM clock
        ipc = ncu_inst_per_cta()
        mhz = clocks.summary().get("sm_mhz") or sm_max_mhz()
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        if not ipc or not mhz or avg_launch_s <= 0:
            return None
        achieved = ipc * step_ctas * args.steps / max(match_n, 1) / avg_launch_s
        peak = 4.0 * sms * float(mhz) * 1e6
        return {"achieved": achieved, "peak": peak, "unit": "warp inst/s", "frac": achieved / peak,
                "note": "warp instructions per CTA from profiles/ncu_summary.json (ncu smsp__inst_executed) x CTAs "
                        "per launch / launch time, vs 4 issue slots per SM per cycle at the sampled SM clock; the "
                        "capture is of strip500 (8,192 descriptors): configs with other descriptor counts run "
                        "more or fewer instructions per CTA, so their figure is only indicative"}

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic (reference generator features.cpp:68-197, seed 7)",
            "config": workload_config(args.config, n_images, avg_desc, rows, resolved),
            "parallelism": (f"one plan sharded over {world} GPU(s) by rows / pairs "
                            "(multigpu.shard_plan), no collective on the data path" if world > 1
                            else "1 GPU, two row slots overlapped"),
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d_all),
                    "d2h_bytes_per_step": int(d2h_all), "ms_per_step": e2e_step_s * 1e3,
                    "step_ms": [round(t * 1e3, 3) for t in e2e_times],
                    "source": "pinned host buffers" + (", matches gathered to rank 0 via shared memory"
                                                       if world > 1 else "")},
            "e2e_pageable": (None if page_ms is None else
                             {"value": n_pairs / (page_ms * 1e-3), "unit": UNIT, "ms_per_step": page_ms,
                              "source": "pageable host buffers (std::vector FeatureSet), H2D via "
                                        "pinned staging slots filled by host threads"}),
            "e2e_files": (None if files_ms is None else
                          {"value": n_pairs / (files_ms * 1e-3), "unit": UNIT, "ms_per_step": files_ms,
                           "source": ".feat files streamed into pinned slots as images upload "
                                     "(bmg_execute_plan_files; page cache warm)"}),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "match_kernel", "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": per_launch_bytes,
                         "avg_launch_ms": avg_launch_s * 1e3,
                         "timing": "CUDA events around each launch on its stream, serial-row pass "
                                   "of the same steps after the timed region"},
            "roofline_secondary": {
                "candidates_per_query": cand_q,
                "popc": {"achieved": popc_per_launch / avg_launch_s if avg_launch_s > 0 else 0.0,
                         "peak": micro.get("popc32_per_s"), "unit": "POPC/s",
                         "frac": (popc_per_launch / avg_launch_s / micro["popc32_per_s"]
                                  if micro.get("popc32_per_s") and avg_launch_s > 0 else None),
                         "note": "32-bit POPC per candidate = 4 at 128 bits; peak: profiles/r2_microbench.json"},
                "issue": issue_roofline(),
                "l2_gather": {"achieved": gather_per_launch / avg_launch_s / 1e9 if avg_launch_s > 0 else 0.0,
                              "peak": micro.get("gather16_l2_gbs"), "unit": "GB/s",
                              "frac": (gather_per_launch / avg_launch_s / 1e9 / micro["gather16_l2_gbs"]
                                       if micro.get("gather16_l2_gbs") and avg_launch_s > 0 else None),
                              "note": "20 B (16 B code + 4 B index) per candidate vs the measured random "
                                      "16-byte L2 gather rate"}},
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items()},
            "results_consistent_e2e_vs_resident": consistent_all,
            "wall_s_timed": t_wall,
            "host_cpu": cpu_model(),
        }
    # CPU baseline + parity: rank 0 at N=1 only (the reference on the same
    # inputs; its match lists against the GPU's)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"], line["parity"] = parity_leg(feats, plan_path, rows, args.config,
                                                              gpu_flat, cores)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": cores,
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0 and world == 1 and not args.no_retrieval:
        try:
            line["retrieval"] = retrieval_leg(bm, m, feats, cores, cpu=not args.no_cpu_baseline)
        except Exception as e:  # noqa: BLE001
            line["retrieval"] = {"unavailable": str(e)}
    if rank == 0 and world > 1:
        gi, go, gm = gpu_flat
        line["parity"] = {"status": "gathered result digest (compare with the N=1 line's result_digest)",
                          "digest_gpu": digest(gi, go, gm), "pairs": int(len(gi)), "matches": int(len(gm))}
    if rank == 0:
        # digest of the whole result (every pair), comparable across N
        gi, go, gm = gpu_flat
        line["result_digest"] = {"digest": digest(gi, go, gm), "pairs": int(len(gi)), "matches": int(len(gm))}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist_barrier()
        dist.destroy_process_group()
    m.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
