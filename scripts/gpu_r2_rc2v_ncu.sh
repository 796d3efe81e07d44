#!/bin/bash
# ncu --set full of the two-iteration kernel in the contracted arithmetic (scaled rotations), L1B_TB=0
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L1B_TB=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fista_rc2v -s 6 -c 1 -o gpurun_out/r2_rc2v_scaled -f \
  python bench.py --steps 20 --no-sparse --no-e2e --no-configs --no-cpu > gpurun_out/ncu_rc2v_scaled.log 2>&1; echo "exit $?" >> gpurun_out/ncu_rc2v_scaled.log
ncu -i gpurun_out/r2_rc2v_scaled.ncu-rep --page details > gpurun_out/r2_ncu_full_fista_rc2v_scaled.txt 2>&1
