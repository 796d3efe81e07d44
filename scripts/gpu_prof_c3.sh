#!/bin/bash
# ncu captures: one cooperative PCG launch of C3 (pdNCG) and the device RNG kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python configs.py --only c3 --no-cpu > gpurun_out/c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_loop -s 3 -c 1 \
  -o gpurun_out/ncu_pcg_loop python configs.py --only c3 --no-cpu > gpurun_out/ncu_pcg.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"pcg_loop|ncg|ls_|dot_|grad|spmv" --csv --log-file gpurun_out/c3_launches.csv python configs.py --only c3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:mt_ -c 4 -o gpurun_out/ncu_rng python scripts/rng_probe.py > gpurun_out/ncu_rng.log 2>&1
