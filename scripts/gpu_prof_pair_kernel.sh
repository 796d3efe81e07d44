#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cd_pair_kernel -c 1 -o gpurun_out/pair_kernel python configs.py --only c2 --no-cpu > gpurun_out/pair_kernel_prof.log 2>&1
echo "exit $?" >> gpurun_out/pair_kernel_prof.log
