#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rng.py -x -q > gpurun_out/pytest_rng.log 2>&1; echo "exit $?" >> gpurun_out/pytest_rng.log
timeout 900 python configs.py --only c5 --c5-ranks 0,3,7 > gpurun_out/c5.log 2>&1; echo "exit $?" >> gpurun_out/c5.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
