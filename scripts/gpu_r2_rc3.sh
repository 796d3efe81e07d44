#!/bin/bash
# three-iteration FISTA kernel: parity tests, smoke, A/B against two iterations per launch, ncu of the kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rc.py tests/test_gpu_fista.py tests/test_gpu_configs.py -k "not c2 and not c3 and not c5" -m gpu -q -x > gpurun_out/pytest_rc3.log 2>&1; echo "exit $?" >> gpurun_out/pytest_rc3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
for rc3 in 1 0 1 0; do
  for k in 20 500; do
    L1B_RC3=$rc3 timeout 300 python bench.py --steps $k --no-sparse --no-e2e --no-configs --no-cpu >> gpurun_out/rc3_ab.log 2>&1
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fista_rc3v -s 3 -c 1 -o gpurun_out/r2_rc3v_fma -f \
  python bench.py --steps 20 --no-sparse --no-e2e --no-configs --no-cpu > gpurun_out/ncu_rc3.log 2>&1; echo "exit $?" >> gpurun_out/ncu_rc3.log
