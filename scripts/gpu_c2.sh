#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pcdm_plan.py tests/test_gpu_solvers.py tests/test_gpu_edges.py -x -q > gpurun_out/pytest_c2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_c2.log
for i in 1 2; do
timeout 600 python configs.py --only c2 --no-cpu > gpurun_out/c2_$i.log 2>&1
L1B_PCDM_PLAN=0 timeout 600 python configs.py --only c2 --no-cpu >> gpurun_out/c2_$i.log 2>&1
done
