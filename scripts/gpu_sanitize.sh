#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family (small sizes)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
SAN=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $SAN --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_smoke.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.log
done
timeout 900 python -m pytest tests/test_gpu_rng.py -k alternating -m gpu -q > gpurun_out/pytest_alt.log 2>&1; echo "exit $?" >> gpurun_out/pytest_alt.log
