#!/bin/bash
# A/B of two builds of libl1b.so (abtest/libl1b_{old,new}.so), alternating, same box.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LIB=paper_1503_03520_b200/lib/libl1b.so
for round in 1 2 3; do
  for v in ${AB_VARIANTS:-old new}; do
    cp abtest/libl1b_$v.so $LIB
    echo "== $v" >> gpurun_out/ab.log
    timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --steps ${AB_STEPS:-40} --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
    echo >> gpurun_out/ab.log
  done
done
cp abtest/libl1b_${AB_FINAL:-new}.so $LIB
