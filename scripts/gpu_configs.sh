#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python configs.py --only c1,c2,c3,c4 --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo "exit $?" >> gpurun_out/configs.log
timeout 900 python configs.py --only c5 --c5-ranks 0,1,2,3,4,5,6,7 --out gpurun_out/c5.json > gpurun_out/c5.log 2>&1; echo "exit $?" >> gpurun_out/c5.log
