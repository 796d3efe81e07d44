#!/bin/bash
# shard tests vs the oracle, IPC peers, run_experiment through the interposer, e2e probe, bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shards.py tests/test_gpu_ipc_peers.py tests/test_gpu_run_experiment.py tests/test_gpu_native_dist.py -m gpu -q > gpurun_out/pytest_b.log 2>&1; echo "exit $?" >> gpurun_out/pytest_b.log
timeout 300 python scripts/e2e_probe.py 500 > gpurun_out/e2e_probe.log 2>&1; echo "exit $?" >> gpurun_out/e2e_probe.log
timeout 900 python bench.py --steps 20 --warmup 4 --no-configs --no-cpu > gpurun_out/bench20.log 2>&1; echo "exit $?" >> gpurun_out/bench20.log
