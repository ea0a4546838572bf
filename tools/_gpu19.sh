#!/bin/bash
out=gpurun_out/r1ad; mkdir -p $out
bash tools/_ab.sh r1ad base d3 d4 base
