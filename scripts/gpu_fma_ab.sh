#!/bin/bash
# A/B of the exact and the contracted (fma) matrix-free FISTA kernels at C4, plus their parity tests
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rc.py -m gpu -q -x > gpurun_out/pytest_rc.log 2>&1; echo "exit $?" >> gpurun_out/pytest_rc.log
for a in exact fma exact fma; do
  for k in 20 500; do
    timeout 300 python bench.py --arith $a --steps $k --no-sparse --no-e2e --no-configs --no-cpu >> gpurun_out/fma_ab.log 2>&1
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fista_rc2v -s 6 -c 1 -o gpurun_out/r2_rc2v_fma -f \
  python bench.py --arith fma --steps 20 --no-sparse --no-e2e --no-configs --no-cpu > gpurun_out/ncu_fma.log 2>&1
