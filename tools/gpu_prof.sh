#!/bin/bash
# Full ncu captures of the hot kernels + a launch list (bench.py workload),
# plus one bench line.  usage: gpurun --timeout 1800 -- bash tools/gpu_prof.sh <tag>
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
for k in match_kernel project_tc_kernel codes_tma_kernel mean_sums_kernel mean_resolve_kernel tables_fused_kernel codes_fixup_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 \
      -o $out/prof_$k $B > $out/ncu_$k.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $out/ncu_launch.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --config pair1 --steps 20 --warmup 5 > $out/bench_pair1.json 2> $out/bench_pair1.err
timeout 900 python bench.py --config strip500 --steps 5 --warmup 3 > $out/bench_strip.json 2> $out/bench_strip.err
timeout 900 python bench.py --config shard16k --steps 5 --warmup 3 > $out/bench_shard16k.json 2> $out/bench_shard16k.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
ls $out
