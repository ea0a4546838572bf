#!/bin/bash
# Full GPU suite + smoke + sanitizers over the kernel-covering subset.
tag=${1:-final}; out=gpurun_out/$tag; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
tail -2 $out/pytest_gpu.log; tail -2 $out/smoke.log
bash tools/sanitize.sh $tag
