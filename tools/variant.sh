#!/bin/bash
# Build an alternative libchp (kernel-variant A/B timing): tools/variant.sh NAME [-DFLAG=V ...]
# -> paper_2304_14074_b200/csrc/build/NAME/libchp_NAME.so  (use with CHP_LIB=...)
set -e
cd "$(dirname "$0")/../paper_2304_14074_b200/csrc"
n=$1; shift
mkdir -p build/$n
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
  --expt-relaxed-constexpr "$@" -c -o build/$n/chp_2d.o chp_2d.cu 2> build/$n/ptxas.txt
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/$n/libchp_$n.so \
  build/chp_api.o build/chp_engine.o build/$n/chp_2d.o build/chp_1d.o build/chp_ddm.o
grep -A2 "linb8k2d_\(rowb\|colb\)ILi1024" build/$n/ptxas.txt | grep -E "spill|Used" || true
