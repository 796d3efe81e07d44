#!/bin/bash
# build_variant.sh NAME "-DFLAG=.. ..." : abtest/libl1b_NAME.so = the library with
# k_iter_rc.cu recompiled under the given defines (A/B runs, scripts/gpu_ab.sh)
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p abtest build/variant_$NAME
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr"
nvcc $FLAGS "$@" -c paper_1503_03520_b200/csrc/k_iter_rc.cu -o build/variant_$NAME/k_iter_rc.o
OBJS=$(ls build/l1b/*.o | grep -v k_iter_rc.o)
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o abtest/libl1b_$NAME.so $OBJS build/variant_$NAME/k_iter_rc.o -lcudart -ldl
echo "abtest/libl1b_$NAME.so"
