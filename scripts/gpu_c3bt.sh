#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L1B_PCG_BT=512 timeout 900 python -m pytest tests/test_gpu_pcg_pair.py tests/test_gpu_solvers.py -x -q > gpurun_out/pytest_c3bt.log 2>&1; echo "exit $?" >> gpurun_out/pytest_c3bt.log
for i in 1 2; do
timeout 600 python configs.py --only c3 --no-cpu > gpurun_out/c3bt_$i.log 2>&1
L1B_PCG_BT=512 timeout 600 python configs.py --only c3 --no-cpu >> gpurun_out/c3bt_$i.log 2>&1
done
