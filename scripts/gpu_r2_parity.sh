#!/bin/bash
# Round 2: full GPU suite (incl. the config-size parity tests) + the reference arm on C4 itself
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 3 ) > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
