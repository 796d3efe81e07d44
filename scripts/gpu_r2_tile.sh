#!/bin/bash
# Tile kernel: full GPU suite, smoke, bench, then the ncu captures (launch list of
# the bench command, --set full of one fista_tb_kernel launch with source)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 20 --no-sparse --no-e2e --no-configs --no-cpu > gpurun_out/bench20.log 2>&1; echo "exit $?" >> gpurun_out/bench20.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench_tile.csv \
  python bench.py --steps 20 --no-sparse --no-e2e --no-configs --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "exit $?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fista_tb_kernel -s 3 -c 1 -o gpurun_out/r2_fista_tb -f \
  python scripts/tile_one.py fma > gpurun_out/ncu_tb.log 2>&1; echo "exit $?" >> gpurun_out/ncu_tb.log
ncu -i gpurun_out/r2_fista_tb.ncu-rep --page details > gpurun_out/r2_ncu_full_fista_tb.txt 2>&1
ncu -i gpurun_out/r2_fista_tb.ncu-rep --page source --csv > gpurun_out/r2_fista_tb_source.csv 2>&1
L1B_SOLVE_TRACE=1 timeout 600 python scripts/e2e_probe.py 500 fma > gpurun_out/e2e_probe.log 2>&1
