#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rng.py tests/test_gpu_pcdm_pair.py tests/test_gpu_pcdm_plan.py tests/test_gpu_solvers.py tests/test_gpu_edges.py -x -q > gpurun_out/pytest_pair.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pair.log
for v in 0; do for i in 1 2 3; do L1B_GEN_VARIANT=$v timeout 600 python configs.py --only c2 --no-cpu > gpurun_out/c2_pair_v${v}_$i.log 2>&1; done; done
for v in 0; do L1B_GEN_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pair_launches_v$v.csv python configs.py --only c2 --no-cpu > gpurun_out/pair_prof.log 2>&1; done
echo "exit $?" >> gpurun_out/pair_prof.log
