#!/bin/bash
# contracted arithmetic unified (scaled rotations in the two-iteration kernel too): full suite, bench lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
for tb in 1 0; do
  echo "== L1B_TB=$tb" >> gpurun_out/unify_ab.log
  L1B_TB=$tb timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 2>&1 | grep -o '"value": [0-9.]*\|"launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/unify_ab.log
  echo >> gpurun_out/unify_ab.log
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --force-dist --steps 500 --warmup 4 --no-cpu > gpurun_out/bench_dist1.log 2>&1; echo "exit $?" >> gpurun_out/bench_dist1.log
timeout 1200 python configs.py --only c5 --out gpurun_out/r2_c5_rank_shards.json > gpurun_out/c5.log 2>&1; echo "exit $?" >> gpurun_out/c5.log
