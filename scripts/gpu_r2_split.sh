#!/bin/bash
# Tile kernel: split-phase exchange / symmetric straddle (fma) / no prefetch A/B; full suite; e2e phases
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
  for v in new split symf nopf; do
    cp abtest/libl1b_$v.so $LIB
    run $v
  done
done
cp abtest/libl1b_split.so $LIB
timeout 600 python -m pytest tests/test_gpu_tile.py -m gpu -q > gpurun_out/pytest_split.log 2>&1; echo "exit $?" >> gpurun_out/pytest_split.log
cp abtest/libl1b_new.so $LIB
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
L1B_SOLVE_TRACE=1 timeout 600 python scripts/e2e_probe.py 500 > gpurun_out/e2e_probe.log 2>&1
