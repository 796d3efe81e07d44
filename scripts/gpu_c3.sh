#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pcg_pair.py tests/test_gpu_solvers.py tests/test_gpu_edges.py -x -q > gpurun_out/pytest_c3.log 2>&1; echo "exit $?" >> gpurun_out/pytest_c3.log
timeout 600 python configs.py --only c3 --no-cpu > gpurun_out/c3.log 2>&1
L1B_PCG_PAIR=0 timeout 600 python configs.py --only c3 --no-cpu >> gpurun_out/c3.log 2>&1
