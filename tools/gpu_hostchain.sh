#!/bin/bash
# host FP64 chain throughput on the GPU box's CPU (tools/probe/host_chain.cpp)
out=gpurun_out/${1:-hc}; mkdir -p $out
for ch in 8 16; do for fl in "-mavx2" "-mavx512f"; do
  g++ -O3 $fl -DCH=$ch -pthread tools/probe/host_chain.cpp -o /tmp/hc || continue
  for T in 4 8 16; do [ $((128 / T)) -ge $ch ] || continue; echo "CH=$ch $fl T=$T"; /tmp/hc 400 $T | tail -2; done
done; done > $out/host_chain.log 2>&1
cat $out/host_chain.log
