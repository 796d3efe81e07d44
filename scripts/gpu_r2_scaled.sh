#!/bin/bash
# Scaled rotations + integer shrink in the tile kernel: FP64 pipe probe, parity, A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
scripts/_build/fp64_pipe_probe > gpurun_out/fp64_pipe_probe.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_tile.py tests/test_gpu_rc.py tests/test_gpu_configs.py -k "tile or fma or c4" -m gpu -q -x > gpurun_out/pytest_scaled.log 2>&1; echo "exit $?" >> gpurun_out/pytest_scaled.log
LIB=paper_1503_03520_b200/lib/libl1b.so
for round in 1 2; do
  for v in lift_fsel lift_ishr scal_fsel scal_ishr; do
    cp abtest/libl1b_$v.so $LIB
    echo "== $v" >> gpurun_out/ab.log
    timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
    echo >> gpurun_out/ab.log
  done
done
cp abtest/libl1b_scal_ishr.so $LIB
