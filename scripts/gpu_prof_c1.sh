#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python configs.py --only c1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fista_pair_small -s 4 -c 1 -o gpurun_out/ncu_pair_small python configs.py --only c1 --no-cpu > /dev/null 2>&1
