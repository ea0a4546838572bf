#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over a GPU-test subset
# that reaches every kernel (mean, projection on the tensor cores, codes,
# fixups, tables, match, compaction, executor streams) and the VLAD encoder
# (SAN_SEL overrides the test selection).
# usage: gpurun --timeout 3000 -- bash tools/sanitize.sh TAG
tag=${1:-san}
out=gpurun_out/$tag; mkdir -p $out
SEL="${SAN_SEL:-tests/test_gpu_retrieval.py tests/test_gpu_codes.py tests/test_gpu_mean.py tests/test_gpu_match.py tests/test_gpu_engine.py tests/test_gpu_overlap.py::test_results_unchanged_with_and_without_hand_off}"
DES="not full_size and not large_train and not 16384"
for tool in memcheck synccheck racecheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest $SEL -q -p no:cacheprovider -k "$DES" -x > $out/$tool.log 2>&1
  echo "$tool rc=$?" >> $out/$tool.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $out/$tool.log | tail -4
done
