#!/bin/bash
# C1-C4 on the GPU beside the reference's CPU solvers on the same configs (full runs; C4: 10 iterations at n=2^27)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nproc; lscpu | grep "Model name"; } > gpurun_out/host_cpu.txt
timeout 2400 python configs.py --only c1,c2,c3,c4 --out gpurun_out/r2_configs.json > gpurun_out/configs.log 2>&1; echo "exit $?" >> gpurun_out/configs.log
