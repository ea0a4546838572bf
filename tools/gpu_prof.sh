#!/bin/bash
# Full ncu captures of the hot kernels of the timed value loop (NVTX range
# "value"), the launch list of that loop, and the bench lines of every config.
# usage: gpurun --timeout 3000 -- bash tools/gpu_prof.sh <tag>
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-files --no-retrieval"
N="--nvtx --nvtx-include value/"
for k in match_kernel project_tc_kernel codes_tma_kernel mean_resolve_kernel tables_fused_kernel compact_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none $N -k regex:$k -c 1 \
      -o $out/prof_$k $B > $out/ncu_$k.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none $N --csv \
    --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-files \
    --no-retrieval > $out/ncu_launch.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --config block32 --steps 10 --warmup 3 > $out/bench_block32.json 2> $out/bench_block32.err
timeout 600 python bench.py --config pair1 --steps 20 --warmup 5 > $out/bench_pair1.json 2> $out/bench_pair1.err
timeout 900 python bench.py --config shard16k --steps 5 --warmup 3 > $out/bench_shard16k.json 2> $out/bench_shard16k.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
ls $out
