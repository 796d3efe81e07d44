#!/bin/bash
# Round-2 numbers for DESIGN / README: default bench (K=500), the driver-style K=20 line, C1-C4 beside the
# reference CPU solvers, the N>1 line at one rank (native NCCL driver), launch list of the bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nproc; lscpu | grep "Model name"; free -g | head -2; } > gpurun_out/host.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench500.log 2>&1; echo "exit $?" >> gpurun_out/bench500.log
timeout 900 python bench.py --steps 20 --warmup 4 --no-cpu > gpurun_out/bench20.log 2>&1; echo "exit $?" >> gpurun_out/bench20.log
timeout 1500 python configs.py --only c1,c2,c3,c4 --out gpurun_out/r2_configs.json > gpurun_out/configs.log 2>&1; echo "exit $?" >> gpurun_out/configs.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --force-dist --steps 500 --warmup 4 > gpurun_out/bench_dist1.log 2>&1; echo "exit $?" >> gpurun_out/bench_dist1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 20 --warmup 4 --no-e2e --no-configs --no-cpu --no-sparse > gpurun_out/ncu_bench.log 2>&1; echo "exit $?" >> gpurun_out/ncu_bench.log
