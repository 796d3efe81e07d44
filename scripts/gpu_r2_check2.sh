#!/bin/bash
# full GPU suite (extended C4-size parity test) + C4 config in both arithmetics
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 1500 python configs.py --only c4 --out gpurun_out/r2_configs_c4.json > gpurun_out/configs_c4.log 2>&1; echo "exit $?" >> gpurun_out/configs_c4.log
