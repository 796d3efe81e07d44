#!/bin/bash
# Tile kernel with 16 entries per lane (255 registers, one 8-warp CTA per SM, tiles of 3840) against 8 per lane
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
  for v in new v16; do
    cp abtest/libl1b_$v.so $LIB
    run $v
  done
done
cp abtest/libl1b_v16.so $LIB
timeout 900 python -m pytest tests/test_gpu_tile.py -m gpu -q > gpurun_out/pytest_v16.log 2>&1; echo "exit $?" >> gpurun_out/pytest_v16.log
cp abtest/libl1b_new.so $LIB
