#!/bin/bash
# native shard driver (NCCL + CUDA graph) at one rank, the N>1 bench line at one rank, e2e breakdown
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_native_dist.py -m gpu -q -x > gpurun_out/pytest_native.log 2>&1; echo "exit $?" >> gpurun_out/pytest_native.log
timeout 300 python scripts/e2e_probe.py 500 > gpurun_out/e2e_probe.log 2>&1; echo "exit $?" >> gpurun_out/e2e_probe.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --force-dist --steps 500 --warmup 4 --no-cpu > gpurun_out/bench_dist1.log 2>&1; echo "exit $?" >> gpurun_out/bench_dist1.log
L1B_NATIVE_DIST=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 1 --force-dist --steps 500 --warmup 4 --no-cpu --no-e2e > gpurun_out/bench_dist1_py.log 2>&1; echo "exit $?" >> gpurun_out/bench_dist1_py.log
