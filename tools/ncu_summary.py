"""Summarise ncu reports (.ncu-rep from `ncu --set full`) and launch lists
(`ncu --metrics gpu__time_duration.sum --csv`) into profiles/.

    python tools/ncu_summary.py --round r1 --match gpurun_out/prof_match.ncu-rep \
        --mean gpurun_out/prof_mean.ncu-rep --codes gpurun_out/prof_codes.ncu-rep \
        --launches gpurun_out/launches.csv

Writes profiles/<round>_ncu_summary.md and profiles/ncu_summary.json (the
latter is read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.per_cycle_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]
UNITS = {"gpu__time_duration.sum": "ms"}


def raw(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = (vals[i], units[i])
    return d


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def launches(path: Path) -> dict:
    text = path.read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        per[name][0] += 1
        per[name][1] += v
    return dict(per)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r1")
    ap.add_argument("--match")
    ap.add_argument("--mean")
    ap.add_argument("--codes")
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[], help="key=path.ncu-rep (any kernel)")
    ap.add_argument("--workload", default="strip500, 3 rows")
    a = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    summary = {}
    md = [f"# ncu summary ({a.round})", "",
          "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
          f"(gpurun), one launch per kernel, bench.py workload ({a.workload}). "
          "ncu times are cold-cache and serialised: compare shares, not absolutes.", ""]
    reps = [("match_kernel", a.match), ("row_mean_tma_kernel", a.mean), ("codes_kernel", a.codes)]
    reps += [tuple(r.split("=", 1)) for r in a.rep]
    for key, rep in reps:
        if not rep:
            continue
        d = raw(Path(rep))
        dram = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
        summary[key] = {"kernel": d["kernel"], "dram_bytes_per_launch": dram,
                        "metrics": {m: v for m, v in d.items() if m != "kernel"}}
        md += [f"## {key}", "", f"`{d['kernel']}`", "", "| metric | value |", "|---|---|"]
        md += [f"| {m} | {v[0]} {v[1]} |" for m, v in d.items() if m != "kernel"]
        md += [f"| dram read+write per launch | {dram / 1e6:.1f} MB |", ""]
    if a.launches:
        per = launches(Path(a.launches))
        total = sum(v[1] for v in per.values())
        summary["launch_list"] = {k: {"launches": v[0], "ms": v[1]} for k, v in per.items()}
        md += ["## launch list (gpu__time_duration.sum)", "", "| kernel | launches | ms | share |",
               "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| {k} | {v[0]} | {v[1]:.3f} | {100 * v[1] / total:.1f}% |")
    (prof / f"{a.round}_ncu_summary.md").write_text("\n".join(md) + "\n")
    (prof / "ncu_summary.json").write_text(json.dumps(summary, indent=1) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
