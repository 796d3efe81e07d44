#!/bin/bash
# Round-2 final validation and numbers: full GPU suite, smoke, default bench (K = 500), the driver-style K = 20
# line, reference arm (bounded), C1-C4 beside the reference CPU solvers, the N > 1 line at one rank, C5 rank shards,
# launch list of the bench command
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nproc; lscpu | grep "Model name"; free -g | head -2; nvidia-smi --query-gpu=name,power.limit,clocks.max.sm --format=csv; } > gpurun_out/host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench500.log 2>&1; echo "exit $?" >> gpurun_out/bench500.log
timeout 900 python bench.py --steps 20 --warmup 4 --no-cpu > gpurun_out/bench20.log 2>&1; echo "exit $?" >> gpurun_out/bench20.log
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_reference_arm.log 2>&1; echo "exit $?" >> gpurun_out/bench_reference_arm.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --force-dist --steps 500 --warmup 4 --no-cpu > gpurun_out/bench_dist1.log 2>&1; echo "exit $?" >> gpurun_out/bench_dist1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 20 --warmup 4 --no-e2e --no-configs --no-cpu --no-sparse > gpurun_out/ncu_bench.log 2>&1; echo "exit $?" >> gpurun_out/ncu_bench.log
timeout 1500 python configs.py --only c1,c2,c3,c4 --out gpurun_out/r2_configs.json > gpurun_out/configs.log 2>&1; echo "exit $?" >> gpurun_out/configs.log
timeout 1200 python configs.py --only c5 --out gpurun_out/r2_c5_rank_shards.json > gpurun_out/c5.log 2>&1; echo "exit $?" >> gpurun_out/c5.log
