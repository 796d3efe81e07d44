#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cd_epoch_plan -s 5 -c 1 \
  -o gpurun_out/ncu_pcdm python configs.py --only c2 --no-cpu > gpurun_out/ncu_pcdm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python configs.py --only c2 --no-cpu > /dev/null 2>&1
