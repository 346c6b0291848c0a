# GPU: panel-blocked diagonal factorization -- full -m gpu suite, c5/c6 bench, phase profiles (v5 12-phase vs new)
set -x
timeout 600 python probes/p2_phases.py c5 probes/libpgpcv_phases_v5.so > gpurun_out/p2_c5_v5.json 2>&1
timeout 600 python probes/p2_phases.py c5 > gpurun_out/p2_c5.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --workload c6 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c6_cv.json 2> gpurun_out/bench_c6_cv.err
timeout 600 python probes/p2_phases.py c6 > gpurun_out/p2_c6.json 2>&1
echo done
