#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L1B_RC2_VARIANT=4 timeout 900 ncu --set full --clock-control none -k regex:fista_rc2c -s 5 -c 1 \
  -o gpurun_out/ncu_rc2c python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 10 --warmup 3 > gpurun_out/ncu_rc2c.log 2>&1
