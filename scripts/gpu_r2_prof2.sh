#!/bin/bash
# ncu --set full of the tile kernel (scaled rotations, integer shrink) + prefetch / 16-warp A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
LIB=paper_1503_03520_b200/lib/libl1b.so
cp $LIB abtest/libl1b_default.so
for round in 1 2; do
  for v in nopf pf w16; do
    cp abtest/libl1b_$v.so $LIB
    echo "== $v" >> gpurun_out/ab.log
    timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
    echo >> gpurun_out/ab.log
  done
done
cp abtest/libl1b_nopf.so $LIB
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fista_tb_kernel -s 3 -c 1 -o gpurun_out/r2_fista_tb2 -f \
  python scripts/tile_one.py fma > gpurun_out/ncu_tb2.log 2>&1; echo "exit $?" >> gpurun_out/ncu_tb2.log
ncu -i gpurun_out/r2_fista_tb2.ncu-rep --page details > gpurun_out/r2_ncu_full_fista_tb2.txt 2>&1
ncu -i gpurun_out/r2_fista_tb2.ncu-rep --page source --csv > gpurun_out/r2_fista_tb2_source.csv 2>&1
cp abtest/libl1b_default.so $LIB
