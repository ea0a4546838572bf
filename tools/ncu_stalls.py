"""Headline metrics + warp-stall samples of one ncu report: python tools/ncu_stalls.py REP"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
keys = ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__bytes_read.sum", "lts__t_sector_hit_rate.pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__grid_size")
for k, x in zip(h, v):
    if k in keys:
        print(f"{k:70s} {x}")
st = [(k, float(x)) for k, x in zip(h, v) if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
      and x.replace('.', '', 1).isdigit()]
tot = sum(x for _, x in st) or 1
for k, x in sorted(st, key=lambda t: -t[1])[:12]:
    print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * x / tot:5.1f}%")
