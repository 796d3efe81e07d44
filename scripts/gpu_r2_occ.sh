#!/bin/bash
# Tile kernel occupancy variants: per-lane accumulators in global memory, 10 / 12-warp tiles at 96 / 80 registers
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
LIB=paper_1503_03520_b200/lib/libl1b.so
run() {
  echo "== $1" >> gpurun_out/ab.log
  timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
  echo >> gpurun_out/ab.log
}
for round in 1 2; do
  for v in new g8 g10 g8x3 g12; do
    cp abtest/libl1b_$v.so $LIB
    run $v
  done
done
for v in g10 g12; do
  cp abtest/libl1b_$v.so $LIB
  timeout 600 python -m pytest tests/test_gpu_tile.py -m gpu -q -x > gpurun_out/pytest_$v.log 2>&1; echo "exit $?" >> gpurun_out/pytest_$v.log
done
cp abtest/libl1b_new.so $LIB
