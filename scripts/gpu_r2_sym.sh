#!/bin/bash
# Tile kernel: symmetric straddle + neighbour mbarriers: parity, A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
timeout 1500 python -m pytest tests/test_gpu_tile.py tests/test_gpu_rc.py tests/test_gpu_configs.py -k "tile or fma or c4" -m gpu -q > gpurun_out/pytest_sym.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sym.log
LIB=paper_1503_03520_b200/lib/libl1b.so
cp $LIB abtest/libl1b_default.so
for round in 1 2; do
  for v in base sym nsync sym_nsync; do
    cp abtest/libl1b_$v.so $LIB
    echo "== $v" >> gpurun_out/ab.log
    timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
    echo >> gpurun_out/ab.log
  done
done
for k in 6 10; do
  echo "== sym_nsync K=$k" >> gpurun_out/ab.log
  L1B_TB_K=$k timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
  echo >> gpurun_out/ab.log
done
cp abtest/libl1b_default.so $LIB
