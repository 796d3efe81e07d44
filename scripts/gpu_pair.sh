#!/bin/bash
# pair-local CD / PCDM: parity tests and the C2 timing (pair path vs direct epochs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pcdm_pair.py tests/test_gpu_pcdm_plan.py tests/test_gpu_solvers.py tests/test_gpu_edges.py -x -q > gpurun_out/pytest_pair.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pair.log
for i in 1 2; do
timeout 600 python configs.py --only c2 --no-cpu > gpurun_out/c2_pair_$i.log 2>&1
L1B_PCDM_PAIR=0 timeout 600 python configs.py --only c2 --no-cpu > gpurun_out/c2_direct_$i.log 2>&1
done
