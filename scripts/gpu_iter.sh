#!/bin/bash
# Tuning call: headline parity tests, a short bench (no sparse / e2e / cpu legs), C5 rank trace.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rc.py tests/test_gpu_fista.py tests/test_gpu_shards.py -x -q > gpurun_out/pytest_iter.log 2>&1; echo "exit $?" >> gpurun_out/pytest_iter.log
for i in 1 2; do timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --steps 200 --warmup 5 >> gpurun_out/bench_iter.log 2>&1; done
L1B_GEN_TRACE=1 timeout 600 python configs.py --only c5 --c5-ranks 3 --c5-iters 40 > gpurun_out/c5_trace.log 2>&1
