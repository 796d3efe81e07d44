#!/bin/bash
# contracted kernels with the rotation as three shears (lifting): parity, A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rc.py tests/test_gpu_native_dist.py tests/test_gpu_configs.py -k "fma or c4 or native" -m gpu -q -x > gpurun_out/pytest_lift.log 2>&1; echo "exit $?" >> gpurun_out/pytest_lift.log
for k in 20 500 20 500; do
  timeout 300 python bench.py --steps $k --no-sparse --no-e2e --no-configs --no-cpu >> gpurun_out/lift_ab.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fista_rc2v -s 6 -c 1 -o gpurun_out/r2_rc2v_lift -f \
  python bench.py --steps 20 --no-sparse --no-e2e --no-configs --no-cpu > gpurun_out/ncu_lift.log 2>&1; echo "exit $?" >> gpurun_out/ncu_lift.log
