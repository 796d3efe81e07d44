#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rc.py -x -q -k "two_iteration" > gpurun_out/pytest_carry.log 2>&1; echo "exit $?" >> gpurun_out/pytest_carry.log
L1B_RC2_VARIANT=4 timeout 900 python -m pytest tests/test_gpu_shards.py tests/test_gpu_fista.py -x -q > gpurun_out/pytest_carry2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_carry2.log
rm -f gpurun_out/ab_env.log
AB_STEPS=500 AB_VARIANTS="0 4" bash scripts/gpu_ab_env.sh
