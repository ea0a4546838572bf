#!/bin/bash
# Build an experimental libbmg variant: tools/build_variant.sh NAME -DMACRO=V ...
# (output paper_2505_22089_b200/libbmg_NAME.so; select with BMG_LIBBMG=<path>)
name=$1; shift
cd "$(dirname "$0")/../paper_2505_22089_b200/csrc"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 \
  -Xcompiler -fPIC,-Wall -shared -cudart static "$@" -o ../libbmg_$name.so \
  $(python3 -c 'import sys; sys.path.insert(0, ".."); import _build; print(" ".join(_build.SOURCES))')
