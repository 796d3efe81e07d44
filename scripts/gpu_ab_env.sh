#!/bin/bash
# A/B of L1B_RC2_VARIANT values on the headline bench (same box, alternating).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
[ -n "$AB_SKIP_TESTS" ] || { timeout 900 python -m pytest tests/test_gpu_rc.py -x -q -k "two_iteration" > gpurun_out/pytest_ab.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ab.log; }
for round in 1 2; do
  for v in ${AB_VARIANTS:-0 4}; do
    echo -n "== $v " >> gpurun_out/ab_env.log
    L1B_RC2_VARIANT=$v timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --steps ${AB_STEPS:-40} --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab_env.log
    echo >> gpurun_out/ab_env.log
  done
done
