#!/bin/bash
# C2 path: parity tests, timing, launch list, ncu full of the epoch kernel and the jump kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pcdm_pair.py tests/test_gpu_pcdm_plan.py tests/test_gpu_rng.py tests/test_gpu_solvers.py tests/test_gpu_configs.py -k "not c3 and not c4 and not c5" -m gpu -q -x > gpurun_out/pytest_c2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_c2.log
timeout 600 python configs.py --only c2 --no-cpu > gpurun_out/c2.log 2>&1; echo "exit $?" >> gpurun_out/c2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python configs.py --only c2 --no-cpu > gpurun_out/ncu_c2.log 2>&1; echo "exit $?" >> gpurun_out/ncu_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cd_pair_kernel|mt_jump_many|cd_mask_scatter|cd_pair_fold|DeviceRadix" -c 8 -o gpurun_out/r2_c2_full -f python configs.py --only c2 --no-cpu > gpurun_out/ncu_c2_full.log 2>&1; echo "exit $?" >> gpurun_out/ncu_c2_full.log
