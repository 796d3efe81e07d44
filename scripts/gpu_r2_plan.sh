cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_bench_line.py tests/test_gpu_rc.py -m gpu -q > gpurun_out/pytest_plan.log 2>&1; echo "exit $?" >> gpurun_out/pytest_plan.log
timeout 900 python bench.py --steps 20 --warmup 4 --no-cpu > gpurun_out/bench20.log 2>&1; echo "exit $?" >> gpurun_out/bench20.log
timeout 600 python bench.py --no-sparse --no-cpu --no-e2e --no-configs --steps 500 --warmup 5 > gpurun_out/bench_tile_final.log 2>&1
