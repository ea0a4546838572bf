out=gpurun_out/r2fin5; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log; tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log; tail -1 $out/smoke.log
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include value/ -k regex:match_kernel -c 1 -o $out/prof_match_kernel python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-files --no-retrieval > $out/ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include value/ --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-files --no-retrieval > $out/l.log 2>&1
ls $out
