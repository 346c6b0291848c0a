set -x
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python probes/p2_phases.py c5 > gpurun_out/p2_c5.json 2>&1
timeout 900 python bench.py --workload c6 --configs-per-step 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c6_cv.json 2> gpurun_out/bench_c6_cv.err
echo done
