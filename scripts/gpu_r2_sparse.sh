#!/bin/bash
# CSR/CSC SpMV (north-star kernels): parity tests, C4 sparse-path timing (burst and K=500), ncu of K1/K2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fista.py tests/test_gpu_solvers.py tests/test_gpu_shards.py -m gpu -q -x > gpurun_out/pytest_sparse.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sparse.log
timeout 900 python bench.py --steps 20 --warmup 4 --no-e2e --no-configs --no-cpu > gpurun_out/bench_sparse20.log 2>&1; echo "exit $?" >> gpurun_out/bench_sparse20.log
timeout 900 python bench.py --steps 500 --warmup 4 --no-e2e --no-configs --no-cpu > gpurun_out/bench_sparse500.log 2>&1; echo "exit $?" >> gpurun_out/bench_sparse500.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 4 -c 2 -o gpurun_out/r2_spmv_full -f python bench.py --steps 4 --warmup 4 --no-e2e --no-configs --no-cpu > gpurun_out/ncu_spmv.log 2>&1; echo "exit $?" >> gpurun_out/ncu_spmv.log
