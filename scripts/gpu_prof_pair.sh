#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_pair -s 3 -c 1 \
  -o gpurun_out/ncu_pcg_pair python configs.py --only c3 --no-cpu > gpurun_out/ncu_pair.log 2>&1
