#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pcdm_pair.py tests/test_gpu_pcdm_plan.py tests/test_gpu_solvers.py tests/test_gpu_edges.py -x -q > gpurun_out/pytest_pair.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pair.log
for i in 1 2; do timeout 600 python configs.py --only c2 --no-cpu > gpurun_out/c2_pair_$i.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pair_launches.csv python configs.py --only c2 --no-cpu > gpurun_out/pair_prof.log 2>&1
echo "exit $?" >> gpurun_out/pair_prof.log
