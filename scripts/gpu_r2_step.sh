#!/bin/bash
# Tile kernel with the store-free step instantiation / merged exchange: parity, bench, K sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
timeout 1500 python -m pytest tests/test_gpu_tile.py tests/test_gpu_rc.py tests/test_gpu_configs.py tests/test_gpu_bench_line.py -k "tile or fma or c4 or line" -m gpu -q > gpurun_out/pytest_step.log 2>&1; echo "exit $?" >> gpurun_out/pytest_step.log
LIB=paper_1503_03520_b200/lib/libl1b.so
run() {
  echo "== $1 K=$2" >> gpurun_out/ab.log
  L1B_TB_K=$2 timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
  echo >> gpurun_out/ab.log
}
for round in 1 2; do
  cp abtest/libl1b_new.so $LIB
  run new 14
  run new 10
  cp abtest/libl1b_k18.so $LIB
  run k18 18
  run k18 14
done
cp abtest/libl1b_new.so $LIB
