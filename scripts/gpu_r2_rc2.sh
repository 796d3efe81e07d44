#!/bin/bash
# Two-iteration kernel with the bit-pattern shrink (old vs new, L1B_TB=0), then the full suite on the new build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
LIB=paper_1503_03520_b200/lib/libl1b.so
run() {
  echo "== $1 (L1B_TB=0)" >> gpurun_out/ab.log
  L1B_TB=0 timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
  echo >> gpurun_out/ab.log
}
for round in 1 2; do
  for v in old new; do
    cp abtest/libl1b_$v.so $LIB
    run $v
  done
done
cp abtest/libl1b_new.so $LIB
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 > gpurun_out/bench_tile_final.log 2>&1
timeout 900 python bench.py --gpus 1 --force-dist --steps 500 --no-cpu > gpurun_out/bench_dist1.log 2>&1; echo "exit $?" >> gpurun_out/bench_dist1.log
