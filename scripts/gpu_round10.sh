set -x
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for w in c3 c5; do timeout 600 python probes/p2_phases.py $w > gpurun_out/p2_$w.json 2>&1; done
timeout 900 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for w in c2 c3 c4; do timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
echo done
