out=gpurun_out/r2j; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
BMG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 2 > $out/bench_n2.json 2> $out/bench_n2.err; echo "n2 rc=$?" >> $out/bench_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-files > $out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 3 -c 1 -o $out/match python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-files > $out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:project_tc_kernel -s 50 -c 1 -o $out/project python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-files > /dev/null 2>&1
ls $out; tail -3 $out/bench.err; tail -5 $out/bench_n2.err
