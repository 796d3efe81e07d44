#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L1B_PCDM_WALK_CHECK=1 timeout 900 python -m pytest tests/test_gpu_pcdm_pair.py -m gpu -q -x > gpurun_out/pytest_walk.log 2>&1; echo "exit $?" >> gpurun_out/pytest_walk.log
