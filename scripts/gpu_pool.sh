set -x
timeout 1500 python -m pytest tests/test_gpu_bisect.py tests/test_gpu_gls.py -x -q > gpurun_out/pytest_pool.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_pool.log
timeout 900 python bench.py --workload c6 --configs-per-step 2 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c6_pool.json 2> gpurun_out/bench_c6_pool.err
echo done
