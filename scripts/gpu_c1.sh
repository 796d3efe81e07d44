#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rc.py tests/test_gpu_fista.py tests/test_gpu_edges.py -x -q > gpurun_out/pytest_c1.log 2>&1; echo "exit $?" >> gpurun_out/pytest_c1.log
timeout 600 python configs.py --only c1 --no-cpu > gpurun_out/c1.log 2>&1
L1B_PAIR_SMALL=1 timeout 600 python configs.py --only c1 --no-cpu >> gpurun_out/c1.log 2>&1
L1B_PAIR_SMALL=0 timeout 600 python configs.py --only c1 --no-cpu >> gpurun_out/c1.log 2>&1
